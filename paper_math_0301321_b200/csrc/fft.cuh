// fft.cuh — in-CTA fp64 FFT building blocks for sm_100a (Stockham autosort, radix <= 16).
//
// Used by the x/y/z passes of the fluid solve ("can be solved
// efficiently with the use of the Fast Fourier Transform algorithm").  A CTA holds a
// batch of pencils in shared memory, one pencil = L complex doubles, element i at
// pencil_base[PAD(i)], PAD(i) = i + i/16 (one spare double2 every 16 elements keeps the
// radix-16 strided stores at <= 2-way bank conflict).  Each pencil is transformed by
// Plan<L>::T threads; every pass loads R elements per job into registers, multiplies by
// the inter-pass twiddles, runs an unrolled register DFT-R, and stores in Stockham order,
// so the result is in natural order.  Twiddles come from a device table
// tw[t] = exp(-2 pi i t / L) (computed with sincospi at context creation).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ibk {

__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n >> 1); }

template <int L>
struct Plan {
  static_assert(L >= 4 && (L & (L - 1)) == 0, "power of two");
  static constexpr int RMAX = L >= 16 ? 16 : L;
  static constexpr int T = L / RMAX;                           // threads per pencil
  static constexpr int NPASS = (ilog2c(L) + 3) / 4;            // passes of radix <= 16
  static constexpr int R0 = L >> (4 * (NPASS - 1));            // first-pass radix
  static constexpr int LD = L + L / 16 + 1;                    // padded pencil stride
  __host__ __device__ static constexpr int radix(int p) { return p == 0 ? R0 : 16; }
  __host__ __device__ static constexpr int ns(int p) { return p == 0 ? 1 : R0 << (4 * (p - 1)); }
};

__device__ __forceinline__ int PAD(int i) { return i + (i >> 4); }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

// cos / sin of 2 pi j / 16 (correctly rounded literals)
#define IBK_C1 0.92387953251128675613
#define IBK_S1 0.38268343236508977173
#define IBK_R2 0.70710678118654752440
__device__ __forceinline__ double cos16(int j) {
  switch (j & 15) {
    case 0: return 1.0;      case 1: return IBK_C1;   case 2: return IBK_R2;   case 3: return IBK_S1;
    case 4: return 0.0;      case 5: return -IBK_S1;  case 6: return -IBK_R2;  case 7: return -IBK_C1;
    case 8: return -1.0;     case 9: return -IBK_C1;  case 10: return -IBK_R2; case 11: return -IBK_S1;
    case 12: return 0.0;     case 13: return IBK_S1;  case 14: return IBK_R2;  default: return IBK_C1;
  }
}
__device__ __forceinline__ double sin16(int j) { return cos16(j - 4); }

// a * exp(SIGN 2 pi i j / 16), j a compile-time constant after unrolling
template <int SIGN>
__device__ __forceinline__ double2 mul_root16(double2 a, int j) {
  j &= 15;
  if (j == 0) return a;
  if (j == 8) return make_double2(-a.x, -a.y);
  if (j == 4) return SIGN > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
  if (j == 12) return SIGN > 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
  if (j == 2 || j == 6 || j == 10 || j == 14) {   // (+-1 +- i)/sqrt 2
    const double c = cos16(j), s = SIGN * sin16(j);
    return make_double2((a.x * c) - (a.y * s), (a.x * s) + (a.y * c));
  }
  const double c = cos16(j), s = SIGN * sin16(j);
  return make_double2(a.x * c - a.y * s, a.x * s + a.y * c);
}

__host__ __device__ constexpr int brev(int i, int bits) {
  return bits == 0 ? 0 : (((i & 1) << (bits - 1)) | brev(i >> 1, bits - 1));
}

// In-register DFT of length R (R | 16): v[k] <- sum_r v[r] exp(SIGN 2 pi i r k / R).
template <int R, int SIGN>
__device__ __forceinline__ void dft_reg(double2 *v) {
  constexpr int B = ilog2c(R);
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int j = (((i & 1) << 3) | ((i & 2) << 1) | ((i & 4) >> 1) | ((i & 8) >> 3)) >> (4 - B);
    if (i < j) { double2 t = v[i]; v[i] = v[j]; v[j] = t; }
  }
#pragma unroll
  for (int st = 0; st < B; ++st) {
#pragma unroll
    for (int bi = 0; bi < R / 2; ++bi) {
      const int half = 1 << st;
      const int k = bi & (half - 1);
      const int s = (bi >> st) << (st + 1);
      double2 a = v[s + k];
      double2 b = mul_root16<SIGN>(v[s + k + half], k * (8 >> st));
      v[s + k] = cadd(a, b);
      v[s + k + half] = csub(a, b);
    }
  }
}

template <int SIGN>
__device__ __forceinline__ double2 twiddle(const double2 *__restrict__ tw, int t) {
  double2 w = __ldg(&tw[t]);
  if (SIGN > 0) w.y = -w.y;
  return w;
}

// One Stockham pass over one pencil by thread t (0 <= t < T).  Caller guarantees all CTA
// threads call it (it contains __syncthreads).
template <int L, int SIGN, int PASS>
__device__ __forceinline__ void fft_pass(double2 *b, int t, const double2 *__restrict__ tw) {
  using P = Plan<L>;
  constexpr int R = P::radix(PASS);
  constexpr int NS = P::ns(PASS);
  constexpr int NR = L / R;
  constexpr int J = NR / P::T;          // jobs per thread
  double2 v[J * R];
#pragma unroll
  for (int q = 0; q < J; ++q) {
    const int j = t + q * P::T;
#pragma unroll
    for (int r = 0; r < R; ++r) v[q * R + r] = b[PAD(j + r * NR)];
  }
#pragma unroll
  for (int q = 0; q < J; ++q) {
    const int j = t + q * P::T;
    if (NS > 1) {
      const int jm = j % NS;
#pragma unroll
      for (int r = 1; r < R; ++r) v[q * R + r] = cmul(v[q * R + r], twiddle<SIGN>(tw, jm * r * (L / (NS * R))));
    }
    dft_reg<R, SIGN>(&v[q * R]);
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < J; ++q) {
    const int j = t + q * P::T;
    const int base = (j / NS) * NS * R + (j % NS);
#pragma unroll
    for (int r = 0; r < R; ++r) b[PAD(base + r * NS)] = v[q * R + r];
  }
  __syncthreads();
}

// Full length-L transform of the pencil at b (natural order in and out).
template <int L, int SIGN>
__device__ __forceinline__ void fft_pencil(double2 *b, int t, const double2 *__restrict__ tw) {
  fft_pass<L, SIGN, 0>(b, t, tw);
  if constexpr (Plan<L>::NPASS > 1) fft_pass<L, SIGN, 1>(b, t, tw);
  if constexpr (Plan<L>::NPASS > 2) fft_pass<L, SIGN, 2>(b, t, tw);
}

}  // namespace ibk
