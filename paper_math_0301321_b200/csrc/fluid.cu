// fluid.cu — step 3 of the IB step on sm_100a: eq:discreteNS1-2
// solved with a hand-written fp64 3-D FFT.
//
//   xfwd : r = rho u/dt - rho sum_k u_k D_k^{+-} u + F   (upwind rule, PAPER.md 676-691)
//          fused with the real-to-complex FFT along x (length-N/2 complex FFT + split);
//          also re-zeroes F for the next spread.
//   ypass: complex FFT along y of every (z, kx) column, in place (forward / inverse).
//   zpass: complex FFT along z, the per-mode implicit-viscosity + projection solve,
//          inverse FFT along z — one kernel, one read and one write of the spectrum.
//   xinv : complex-to-real FFT along x, writes u^{n+1}; flags non-finite values.
//
// Spectrum layout: [comp][z][y][kx] with kx in [0, N/2], row pitch P = N/2 + 2 complex
// (32-byte aligned rows).  All transforms are unnormalised; the 1/N^3 of the inverse is
// folded into the per-mode solve.
#include <climits>

#include "fft.cuh"
#include "ib_internal.cuh"

namespace ibk {

// ------------------------------------------------------------------ tile configuration
template <int N> struct XCfg {      // x passes: RB rows of one z-plane per CTA
  static constexpr int M = N / 2;
  static constexpr int T = Plan<M>::T;
  static constexpr int RB = (64 / T) < N ? (64 / T) : N;
};
template <int N> struct YCfg {      // y pass: C consecutive kx columns per CTA
  static constexpr int T = Plan<N>::T;
  static constexpr int C0 = 128 / T;
  static constexpr int C = C0 < 8 ? 8 : (C0 > 32 ? 32 : C0);
};
template <int N> struct ZCfg {      // z pass: C consecutive kx columns x 3 components per CTA
  static constexpr int T = Plan<N>::T;
  static constexpr int C0 = 128 / T;
  static constexpr int C = C0 < 4 ? 4 : (C0 > 32 ? 32 : C0);
};

__device__ __forceinline__ long long step_of(const long long *dev_n, long long n) {
  return dev_n ? *dev_n : n;
}

// ------------------------------------------------------------------ tables
__global__ void k_init_tables(double2 *twN, int N, double2 *twM, int M, double *s, double *l,
                              double h) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < N) {
    double sn, cs;
    sincospi(2.0 * (double)t / (double)N, &sn, &cs);
    twN[t] = make_double2(cs, -sn);                       // exp(-2 pi i t / N)
    // D0 symbol s = sin(2 pi k'/N)/h with signed k'; exactly 0 where 2k = 0 mod N (Z22)
    const int ks = t > N / 2 ? t - N : t;
    s[t] = ((2 * t) % N == 0) ? 0.0 : sinpi(2.0 * (double)ks / (double)N) / h;
    const double sh = sinpi((double)t / (double)N);
    l[t] = 4.0 * sh * sh / (h * h);                       // -symbol of D+D-
  }
  if (t < M) {
    double sn, cs;
    sincospi(2.0 * (double)t / (double)M, &sn, &cs);
    twM[t] = make_double2(cs, -sn);
  }
}

cudaError_t init_tables(ib_ctx *c) {
  const int N = c->g.N;
  k_init_tables<<<(N + 127) / 128, 128, 0, c->stream>>>(c->twN, N, c->twM, N / 2, c->sym_s,
                                                        c->sym_l, c->g.h);
  c->launches++;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ x forward
// MODE 0: step (r from u, F; zero F; FFT); 1: r only -> r_out; 2: FFT of `in` (1 comp).
template <int N, int MODE>
__global__ void __launch_bounds__(3 * XCfg<N>::RB * XCfg<N>::T)
k_xfwd(FluidGeom g, const double *__restrict__ u, double *F, const double *__restrict__ in,
       double *r_out, double2 *spec, const double2 *__restrict__ twN,
       const double2 *__restrict__ twM) {
  constexpr int M = N / 2, RB = XCfg<N>::RB, T = XCfg<N>::T, LD = Plan<M>::LD;
  constexpr int NC = MODE == 2 ? 1 : 3;
  extern __shared__ double2 sm[];
  const int z = blockIdx.y, y0 = blockIdx.x * RB;
  const size_t V = (size_t)N * N * N;
  const double cu = g.rho / g.dt, ra = g.rho * g.invh;

  for (int idx = threadIdx.x; idx < RB * N; idx += blockDim.x) {
    const int row = idx / N, x = idx % N, y = y0 + row;
    const size_t c0 = ((size_t)z * N + y) * N + x;
    double r[3];
    if (MODE == 2) {
      r[0] = in[c0];
    } else {
      const size_t nm[3] = {((size_t)z * N + y) * N + ((x + N - 1) & (N - 1)),
                            ((size_t)z * N + ((y + N - 1) & (N - 1))) * N + x,
                            ((size_t)((z + N - 1) & (N - 1)) * N + y) * N + x};
      const size_t np_[3] = {((size_t)z * N + y) * N + ((x + 1) & (N - 1)),
                             ((size_t)z * N + ((y + 1) & (N - 1))) * N + x,
                             ((size_t)((z + 1) & (N - 1)) * N + y) * N + x};
      double uc[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) uc[k] = __ldg(&u[k * V + c0]);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double *ui = u + i * V;
        double adv = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          // u_k D_k^- if u_k > 0, u_k D_k^+ if u_k < 0 (backward at u_k = 0, Z5)
          const double d = uc[k] < 0.0 ? (__ldg(&ui[np_[k]]) - uc[i]) : (uc[i] - __ldg(&ui[nm[k]]));
          adv += uc[k] * d;
        }
        double Fi = F[i * V + c0];
        r[i] = cu * uc[i] - ra * adv + Fi;
        if (MODE == 0 && Fi != 0.0) F[i * V + c0] = 0.0;
      }
    }
    if (MODE == 1) {
#pragma unroll
      for (int i = 0; i < 3; ++i) r_out[i * V + c0] = r[i];
    } else {
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        double *p = reinterpret_cast<double *>(sm + (i * RB + row) * LD + PAD(x >> 1));
        p[x & 1] = r[i];
      }
    }
  }
  if (MODE == 1) return;
  __syncthreads();
  {
    const int pencil = threadIdx.x / T, t = threadIdx.x % T;
    fft_pencil<M, -1>(sm + pencil * LD, t, twM);
  }
  // split the length-M transform Z of z_n = r_2n + i r_2n+1 into X_k, k = 0..M:
  // E = (Z_k + conj Z_{M-k})/2, O = -i (Z_k - conj Z_{M-k})/2, X_k = E + w^k O,
  // X_{M-k} = conj(E - w^k O), w = exp(-2 pi i/N).
  constexpr int H = M / 2 + 1;
  for (int idx = threadIdx.x; idx < NC * RB * H; idx += blockDim.x) {
    const int pencil = idx / H, k = idx % H;
    const int comp = pencil / RB, row = pencil % RB;
    const double2 Zk = sm[pencil * LD + PAD(k)];
    const double2 Zm = sm[pencil * LD + PAD((M - k) & (M - 1))];
    const double2 E = make_double2(0.5 * (Zk.x + Zm.x), 0.5 * (Zk.y - Zm.y));
    const double2 O = make_double2(0.5 * (Zk.y + Zm.y), -0.5 * (Zk.x - Zm.x));
    const double2 wO = cmul(__ldg(&twN[k]), O);
    double2 *out = spec + (((size_t)comp * N + z) * N + (y0 + row)) * g.P;
    out[k] = cadd(E, wO);
    if (k != M - k) out[M - k] = cconj(csub(E, wO));
  }
}

template <int N>
static cudaError_t launch_xfwd_n(const FluidGeom &g, int mode, const double *u, double *F,
                                 const double *in, double *r_out, double2 *spec, int ncomp,
                                 const double2 *twN, const double2 *twM, cudaStream_t s) {
  using X = XCfg<N>;
  dim3 grid(N / X::RB, N);
  const int nc = mode == 2 ? 1 : 3;
  const size_t smem = (size_t)nc * X::RB * Plan<N / 2>::LD * sizeof(double2);
  const int threads = nc * X::RB * X::T;
  (void)ncomp;
  if (mode == 0)
    k_xfwd<N, 0><<<grid, threads, smem, s>>>(g, u, F, in, r_out, spec, twN, twM);
  else if (mode == 1)
    k_xfwd<N, 1><<<grid, threads, 0, s>>>(g, u, F, in, r_out, spec, twN, twM);
  else
    k_xfwd<N, 2><<<grid, threads, smem, s>>>(g, u, F, in, r_out, spec, twN, twM);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ y pass
template <int N, int SIGN>
__global__ void __launch_bounds__(YCfg<N>::C * YCfg<N>::T)
k_ypass(FluidGeom g, double2 *spec, const double2 *__restrict__ twN) {
  constexpr int C = YCfg<N>::C, T = YCfg<N>::T, LD = Plan<N>::LD, M = N / 2;
  extern __shared__ double2 sm[];
  const int col0 = blockIdx.x * C, z = blockIdx.y, comp = blockIdx.z;
  double2 *base = spec + ((size_t)comp * N + z) * N * g.P;
  for (int idx = threadIdx.x; idx < C * N; idx += blockDim.x) {
    const int y = idx / C, col = idx % C, kx = col0 + col;
    sm[col * LD + PAD(y)] = kx <= M ? base[(size_t)y * g.P + kx] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  fft_pencil<N, SIGN>(sm + (threadIdx.x / T) * LD, threadIdx.x % T, twN);
  for (int idx = threadIdx.x; idx < C * N; idx += blockDim.x) {
    const int y = idx / C, col = idx % C, kx = col0 + col;
    if (kx <= M) base[(size_t)y * g.P + kx] = sm[col * LD + PAD(y)];
  }
}

template <int N>
static cudaError_t launch_ypass_n(const FluidGeom &g, int sign, double2 *spec, int ncomp,
                                  const double2 *twN, cudaStream_t s) {
  using Y = YCfg<N>;
  dim3 grid((N / 2 + 1 + Y::C - 1) / Y::C, N, ncomp);
  const size_t smem = (size_t)Y::C * Plan<N>::LD * sizeof(double2);
  if (sign < 0)
    k_ypass<N, -1><<<grid, Y::C * Y::T, smem, s>>>(g, spec, twN);
  else
    k_ypass<N, +1><<<grid, Y::C * Y::T, smem, s>>>(g, spec, twN);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ z pass + solve
// Per mode k (DESIGN.md §2 S3c):  d = rho/dt + mu (l(kx) + l(ky) + l(kz)),
//   u^ = (r^ - s (s.r^)/|s|^2) / (d N^3),   p^ = -i (s.r^)/|s|^2 / N^3,
//   and on the 8 null modes (every k_a in {0, N/2}): u^ = r^/(d N^3), p^ = 0.
template <int N, int MODE, bool PRESS>
__global__ void __launch_bounds__((PRESS ? 4 : 3) * ZCfg<N>::C * ZCfg<N>::T)
k_zpass(FluidGeom g, double2 *spec, double2 *pspec, const double2 *__restrict__ twN,
        const double *__restrict__ sym_s, const double *__restrict__ sym_l) {
  constexpr int C = ZCfg<N>::C, T = ZCfg<N>::T, LD = Plan<N>::LD, M = N / 2;
  extern __shared__ double2 sm[];
  const int col0 = blockIdx.x * C, ky = blockIdx.y;
  const size_t cstride = (size_t)N * N * g.P, zstride = (size_t)N * g.P;
  double2 *base = spec + (size_t)ky * g.P;
  for (int idx = threadIdx.x; idx < 3 * C * N; idx += blockDim.x) {
    const int comp = idx / (C * N), rem = idx % (C * N);
    const int zz = rem / C, col = rem % C, kx = col0 + col;
    sm[(comp * C + col) * LD + PAD(zz)] =
        kx <= M ? base[comp * cstride + zz * zstride + kx] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const int pencil = threadIdx.x / T, t = threadIdx.x % T;
  fft_pencil<N, -1>(sm + pencil * LD, t, twN);
  if (MODE == 0) {
    const double sy = sym_s[ky], ly = sym_l[ky];
    const bool ny = (ky == 0) || (ky == M);
    const double invV = 1.0 / ((double)N * (double)N * (double)N);
    for (int idx = threadIdx.x; idx < C * N; idx += blockDim.x) {
      const int col = idx / N, kz = idx % N, kx = col0 + col;
      if (kx > M) continue;
      const double sx = sym_s[kx], sz = sym_s[kz];
      const double d = g.rho / g.dt + g.mu * (sym_l[kx] + ly + sym_l[kz]);
      const double inv = invV / d;
      double2 *q0 = sm + (0 * C + col) * LD + PAD(kz);
      double2 *q1 = sm + (1 * C + col) * LD + PAD(kz);
      double2 *q2 = sm + (2 * C + col) * LD + PAD(kz);
      const double2 r0 = *q0, r1 = *q1, r2 = *q2;
      const bool nul = ny && (kx == 0 || kx == M) && (kz == 0 || kz == M);
      if (nul) {
        *q0 = cscale(r0, inv); *q1 = cscale(r1, inv); *q2 = cscale(r2, inv);
        if (PRESS) sm[(3 * C + col) * LD + PAD(kz)] = make_double2(0.0, 0.0);
      } else {
        const double s2 = sx * sx + sy * sy + sz * sz;
        const double2 sr = make_double2(sx * r0.x + sy * r1.x + sz * r2.x,
                                        sx * r0.y + sy * r1.y + sz * r2.y);
        const double2 q = make_double2(sr.x / s2, sr.y / s2);
        *q0 = make_double2((r0.x - sx * q.x) * inv, (r0.y - sx * q.y) * inv);
        *q1 = make_double2((r1.x - sy * q.x) * inv, (r1.y - sy * q.y) * inv);
        *q2 = make_double2((r2.x - sz * q.x) * inv, (r2.y - sz * q.y) * inv);
        if (PRESS) sm[(3 * C + col) * LD + PAD(kz)] = make_double2(q.y * invV, -q.x * invV);
      }
    }
    __syncthreads();
    fft_pencil<N, +1>(sm + pencil * LD, t, twN);
  }
  for (int idx = threadIdx.x; idx < 3 * C * N; idx += blockDim.x) {
    const int comp = idx / (C * N), rem = idx % (C * N);
    const int zz = rem / C, col = rem % C, kx = col0 + col;
    if (kx <= M) base[comp * cstride + zz * zstride + kx] = sm[(comp * C + col) * LD + PAD(zz)];
  }
  if (PRESS) {
    double2 *pb = pspec + (size_t)ky * g.P;
    for (int idx = threadIdx.x; idx < C * N; idx += blockDim.x) {
      const int zz = idx / C, col = idx % C, kx = col0 + col;
      if (kx <= M) pb[zz * zstride + kx] = sm[(3 * C + col) * LD + PAD(zz)];
    }
  }
}

template <int N>
static cudaError_t launch_zpass_n(const FluidGeom &g, int mode, double2 *spec, double2 *pspec,
                                  const double2 *twN, const double *s_, const double *l_,
                                  cudaStream_t s) {
  using Z = ZCfg<N>;
  dim3 grid((N / 2 + 1 + Z::C - 1) / Z::C, N);
  const size_t smem3 = (size_t)3 * Z::C * Plan<N>::LD * sizeof(double2);
  const size_t smem4 = (size_t)4 * Z::C * Plan<N>::LD * sizeof(double2);
  if (mode == 1)
    k_zpass<N, 1, false><<<grid, 3 * Z::C * Z::T, smem3, s>>>(g, spec, pspec, twN, s_, l_);
  else if (pspec)
    k_zpass<N, 0, true><<<grid, 4 * Z::C * Z::T, smem4, s>>>(g, spec, pspec, twN, s_, l_);
  else
    k_zpass<N, 0, false><<<grid, 3 * Z::C * Z::T, smem3, s>>>(g, spec, pspec, twN, s_, l_);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ x inverse (C2R)
// From X_k (k = 0..M) rebuild Z'_k = A + i c B, Z'_{M-k} = conj(A - i c B) with
// A = X_k + conj X_{M-k}, B = X_k - conj X_{M-k}, c = exp(+2 pi i k/N); then the inverse
// length-M FFT of Z' is N (r_even + i r_odd).
template <int N>
__global__ void __launch_bounds__(3 * XCfg<N>::RB * XCfg<N>::T)
k_xinv(FluidGeom g, const double2 *__restrict__ spec, double *out, int ncomp,
       const double2 *__restrict__ twN, const double2 *__restrict__ twM, long long *flag,
       const long long *dev_n, long long n) {
  constexpr int M = N / 2, RB = XCfg<N>::RB, T = XCfg<N>::T, LD = Plan<M>::LD;
  constexpr int H = M / 2 + 1;
  extern __shared__ double2 sm[];
  const int z = blockIdx.y, y0 = blockIdx.x * RB;
  for (int idx = threadIdx.x; idx < ncomp * RB * H; idx += blockDim.x) {
    const int pencil = idx / H, k = idx % H;
    const int comp = pencil / RB, row = pencil % RB;
    const double2 *in = spec + (((size_t)comp * N + z) * N + (y0 + row)) * g.P;
    double2 Xk = in[k], Xm = in[M - k];
    if (k == 0) { Xk.y = 0.0; Xm.y = 0.0; }      // X_0, X_{N/2} are real
    const double2 A = make_double2(Xk.x + Xm.x, Xk.y - Xm.y);
    const double2 B = make_double2(Xk.x - Xm.x, Xk.y + Xm.y);
    const double2 cB = cmul(cconj(__ldg(&twN[k])), B);
    const double2 icB = make_double2(-cB.y, cB.x);
    sm[pencil * LD + PAD(k)] = cadd(A, icB);
    if (k != 0 && k != M - k) sm[pencil * LD + PAD(M - k)] = cconj(csub(A, icB));
  }
  __syncthreads();
  {  // blockDim = ncomp * RB * T: every thread owns a pencil (launcher guarantees)
    const int pencil = threadIdx.x / T, t = threadIdx.x % T;
    fft_pencil<M, +1>(sm + pencil * LD, t, twM);
  }
  bool bad = false;
  const size_t V = (size_t)N * N * N;
  for (int idx = threadIdx.x; idx < ncomp * RB * N; idx += blockDim.x) {
    const int pencil = idx / N, x = idx % N;
    const int comp = pencil / RB, row = pencil % RB;
    const double2 v = sm[pencil * LD + PAD(x >> 1)];
    const double val = (x & 1) ? v.y : v.x;
    bad |= !isfinite(val);
    out[comp * V + ((size_t)z * N + (y0 + row)) * N + x] = val;
  }
  if (flag && __syncthreads_or(bad) && threadIdx.x == 0) {
    const long long st = dev_n ? *dev_n - 1 : n;
    atomicMin(flag, st);
  }
}

template <int N>
static cudaError_t launch_xinv_n(const FluidGeom &g, const double2 *spec, double *out,
                                 int ncomp, const double2 *twN, const double2 *twM,
                                 long long *flag, const long long *dev_n, long long n,
                                 cudaStream_t s) {
  using X = XCfg<N>;
  dim3 grid(N / X::RB, N);
  const size_t smem = (size_t)ncomp * X::RB * Plan<N / 2>::LD * sizeof(double2);
  k_xinv<N><<<grid, ncomp * X::RB * X::T, smem, s>>>(g, spec, out, ncomp, twN, twM, flag,
                                                     dev_n, n);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ dispatch
#define IBK_DISPATCH_N(N_, CALL)                                           \
  switch (N_) {                                                            \
    case 8: return CALL(8);                                                \
    case 16: return CALL(16);                                              \
    case 32: return CALL(32);                                              \
    case 64: return CALL(64);                                              \
    case 128: return CALL(128);                                            \
    case 256: return CALL(256);                                            \
    case 512: return CALL(512);                                            \
    default: return cudaErrorInvalidValue;                                 \
  }

cudaError_t launch_xfwd(const FluidGeom &g, int mode, const double *u, double *F,
                        const double *in, double *r_out, double2 *spec, int ncomp,
                        const double2 *twN, const double2 *twM, cudaStream_t s) {
#define CALL(n) launch_xfwd_n<n>(g, mode, u, F, in, r_out, spec, ncomp, twN, twM, s)
  IBK_DISPATCH_N(g.N, CALL)
#undef CALL
}

cudaError_t launch_ypass(const FluidGeom &g, int sign, double2 *spec, int ncomp,
                         const double2 *twN, cudaStream_t s) {
#define CALL(n) launch_ypass_n<n>(g, sign, spec, ncomp, twN, s)
  IBK_DISPATCH_N(g.N, CALL)
#undef CALL
}

cudaError_t launch_zpass(const FluidGeom &g, int mode, double2 *spec, double2 *pspec,
                         const double2 *twN, const double *sym_s, const double *sym_l,
                         cudaStream_t s) {
#define CALL(n) launch_zpass_n<n>(g, mode, spec, pspec, twN, sym_s, sym_l, s)
  IBK_DISPATCH_N(g.N, CALL)
#undef CALL
}

cudaError_t launch_xinv(const FluidGeom &g, const double2 *spec, double *out, int ncomp,
                        const double2 *twN, const double2 *twM, long long *flag,
                        const long long *dev_n, long long n, cudaStream_t s) {
#define CALL(n_) launch_xinv_n<n_>(g, spec, out, ncomp, twN, twM, flag, dev_n, n, s)
  IBK_DISPATCH_N(g.N, CALL)
#undef CALL
}

template <int N>
static cudaError_t set_attrs_n() {
  const int big = 200 * 1024;
  cudaError_t e = cudaSuccess;
#define SETA(K) if (e == cudaSuccess) e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, big)
  SETA((k_xfwd<N, 0>)); SETA((k_xfwd<N, 2>));
  SETA((k_ypass<N, -1>)); SETA((k_ypass<N, +1>));
  SETA((k_zpass<N, 0, false>)); SETA((k_zpass<N, 0, true>)); SETA((k_zpass<N, 1, false>));
  SETA(k_xinv<N>);
#undef SETA
  return e;
}

cudaError_t fluid_setup_attributes(int N) {
#define CALL(n) set_attrs_n<n>()
  IBK_DISPATCH_N(N, CALL)
#undef CALL
}

}  // namespace ibk
