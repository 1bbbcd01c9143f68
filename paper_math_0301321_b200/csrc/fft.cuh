// fft.cuh — in-CTA fp64 FFT building blocks for sm_100a (Stockham autosort, radix <= 16).
//
// Used by the x/y/z passes of the fluid solve ("can be solved
// efficiently with the use of the Fast Fourier Transform algorithm").  A CTA holds a
// batch of pencils in shared memory, one pencil = L complex doubles, element i at
// pencil_base[PAD(i)] with the XOR swizzle PAD(i) = i ^ (((i >> 1) ^ (i >> 4)) & 7): a
// 16-byte access is served per quarter-warp (8 lanes), and for every pass of every plan
// here (radix-R0 strided stores, contiguous loads) 8 consecutive jobs then fall in 8
// distinct 16-byte bank groups (checked exhaustively for L = 8..1024).  Pencil stride
// LD = L + 1 (odd) keeps 8 different pencils at the same element conflict-free too.  Each pencil is transformed by
// Plan<L>::T threads; every pass loads R elements per job into registers, multiplies by
// the inter-pass twiddles, runs an unrolled register DFT-R, and stores in Stockham order,
// so the result is in natural order.  Twiddles come from a device table
// tw[t] = exp(-2 pi i t / L) (computed with sincospi at context creation).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace ibk {

__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n >> 1); }

template <int L>
struct Plan {
  static_assert(L >= 4 && (L & (L - 1)) == 0, "power of two");
  static constexpr int RMAX = L >= 16 ? 16 : L;
  static constexpr int T = L / RMAX;                           // threads per pencil
  static constexpr int NPASS = (ilog2c(L) + 3) / 4;            // passes of radix <= 16
  static constexpr int R0 = L >> (4 * (NPASS - 1));            // first-pass radix
  static constexpr int LD = L + 1;                             // pencil stride (odd)
  __host__ __device__ static constexpr int radix(int p) { return p == 0 ? R0 : 16; }
  __host__ __device__ static constexpr int ns(int p) { return p == 0 ? 1 : R0 << (4 * (p - 1)); }
};

__device__ __forceinline__ int PAD(int i) { return i ^ (((i >> 1) ^ (i >> 4)) & 7); }

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
  double2 w = __ldg(&tw[t]);         // device table (read-only path)
  if (SIGN > 0) w.y = -w.y;
  return w;
}
// A twiddle table staged in shared memory (persistent kernels that keep it per CTA).
struct SmemTw { const double2 *p; };
template <int SIGN>
__device__ __forceinline__ double2 twiddle(SmemTw tw, int t) {
  double2 w = tw.p[t];
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

// ---------------------------------------------------------------- load/store-functor passes
// The same Stockham passes with the first pass reading through `ld(e)` (e.g. straight from
// HBM into registers: RMAX independent loads per thread) and the last pass writing through
// `st(e, v)` (e.g. straight to HBM), so a 2-pass transform makes ONE shared-memory round
// trip.  The last pass is thread-local in place (it reads and writes positions j + r*NS),
// so results may be stored back into the same pencil without a barrier.
template <int L, int PASS>
struct PassI {
  using P = Plan<L>;
  static constexpr int R = P::radix(PASS), NS = P::ns(PASS), NR = L / R, J = NR / P::T;
};

// v[r] *= w^(e0 r), r = 1..15, w = exp(SIGN 2 pi i / L), from the four table entries
// w^e0, w^2e0, w^4e0, w^8e0 and 11 complex products (each power at most three roundings
// from the table) instead of 15 table reads: the reads' latency (L1 for the global table,
// shared for a staged one) was the largest stall of the column passes.
template <int L, int SIGN, class TW>
__device__ __forceinline__ void twiddle16_pow(double2 *v, int e0, TW tw) {
  const double2 b0 = twiddle<SIGN>(tw, e0), b1 = twiddle<SIGN>(tw, 2 * e0),
                b2 = twiddle<SIGN>(tw, 4 * e0), b3 = twiddle<SIGN>(tw, 8 * e0);
  const double2 p3 = cmul(b0, b1), p12 = cmul(b3, b2);
  v[1] = cmul(v[1], b0);             v[2] = cmul(v[2], b1);
  v[3] = cmul(v[3], p3);             v[4] = cmul(v[4], b2);
  v[5] = cmul(v[5], cmul(b2, b0));   v[6] = cmul(v[6], cmul(b2, b1));
  v[7] = cmul(v[7], cmul(b2, p3));   v[8] = cmul(v[8], b3);
  v[9] = cmul(v[9], cmul(b3, b0));   v[10] = cmul(v[10], cmul(b3, b1));
  v[11] = cmul(v[11], cmul(b3, p3)); v[12] = cmul(v[12], p12);
  v[13] = cmul(v[13], cmul(p12, b0)); v[14] = cmul(v[14], cmul(p12, b1));
  v[15] = cmul(v[15], cmul(p12, p3));
}

// POW: radix-16 passes take their twiddles from twiddle16_pow (4 table reads + products)
// instead of 15 table reads; chosen per kernel by measurement (it frees the latency-bound
// x forward and z passes, but costs the register-heavy y passes more than it saves).
// The 15 twiddles of a thread's radix-16 job held in registers for the kernel's lifetime
// (column passes whose pass-1 job index is the thread's own t, so the set never changes).
struct RegTw16 {
  double2 w[16];
};
template <class T> struct is_regtw : std::false_type {};
template <> struct is_regtw<RegTw16> : std::true_type {};
// w[r] = exp(SIGN 2 pi i e0 r / L) from a device table tw[t] = exp(-2 pi i t / L)
template <int SIGN>
__device__ __forceinline__ RegTw16 make_regtw16(const double2 *__restrict__ tw, int e0) {
  RegTw16 r;
  r.w[0] = make_double2(1.0, 0.0);
#pragma unroll
  for (int k = 1; k < 16; ++k) r.w[k] = twiddle<SIGN>(tw, e0 * k);
  return r;
}

template <int L, int SIGN, int PASS, bool POW = false, class TW, class LDF>
__device__ __forceinline__ void pass_lc(double2 *v, int t, TW tw, LDF ld) {
  using I = PassI<L, PASS>;
#pragma unroll
  for (int q = 0; q < I::J; ++q) {
    const int j = t + q * Plan<L>::T;
#pragma unroll
    for (int r = 0; r < I::R; ++r) {
      if constexpr (std::is_invocable_v<LDF, int, int>)
        v[q * I::R + r] = ld(j + r * I::NR, q * I::R + r);     // (element, pass-0 slot)
      else
        v[q * I::R + r] = ld(j + r * I::NR);
    }
  }
#pragma unroll
  for (int q = 0; q < I::J; ++q) {
    const int j = t + q * Plan<L>::T;
    if (I::NS > 1) {
      const int jm = j % I::NS;
      if constexpr (is_regtw<TW>::value) {
#pragma unroll
        for (int r = 1; r < I::R; ++r) v[q * I::R + r] = cmul(v[q * I::R + r], tw.w[r]);
      } else if constexpr (I::R == 16 && POW) {
        twiddle16_pow<L, SIGN>(&v[q * I::R], jm * (L / (I::NS * I::R)), tw);
      } else {
#pragma unroll
        for (int r = 1; r < I::R; ++r)
          v[q * I::R + r] = cmul(v[q * I::R + r], twiddle<SIGN>(tw, jm * r * (L / (I::NS * I::R))));
      }
    }
    dft_reg<I::R, SIGN>(&v[q * I::R]);
  }
}

template <int L, int PASS, class STF>
__device__ __forceinline__ void pass_st(const double2 *v, int t, STF st) {
  using I = PassI<L, PASS>;
#pragma unroll
  for (int q = 0; q < I::J; ++q) {
    const int j = t + q * Plan<L>::T;
    const int base = (j / I::NS) * I::NS * I::R + (j % I::NS);
#pragma unroll
    for (int r = 0; r < I::R; ++r) st(base + r * I::NS, v[q * I::R + r]);
  }
}

// Length-L transform of one pencil by its T threads: pass 0 reads via ld, the last pass
// writes via st, intermediate passes exchange through the padded smem pencil sp.
// LD_SMEM: ld reads sp itself (a barrier then separates pass-0 loads from stores).
// WARP: the pencil's T threads are consecutive lanes of one warp (T <= 32, thread index
// t-fastest), so exchanges need only __syncwarp; otherwise every thread of the CTA must
// call this (it contains __syncthreads when NPASS > 1).
template <bool WARP>
__device__ __forceinline__ void pencil_sync() {
  if (WARP) __syncwarp(); else __syncthreads();
}

struct NoOp {
  __device__ __forceinline__ void operator()() const {}
};

template <int L, int SIGN, bool LD_SMEM, bool WARP, bool POW = false, class LDF, class STF,
          class AF = NoOp>
__device__ __forceinline__ void fft_io(double2 *sp, int t, const double2 *__restrict__ tw,
                                       LDF ld, STF st, AF after_load = AF()) {
  using P = Plan<L>;
  static_assert(!WARP || (P::T <= 32), "pencil must fit in a warp");
  double2 v[P::RMAX];
  auto sst = [sp](int e, double2 x) { sp[PAD(e)] = x; };
  auto sld = [sp](int e) { return sp[PAD(e)]; };
  pass_lc<L, SIGN, 0>(v, t, tw, ld);
  after_load();      // pass-0 inputs are in registers: e.g. start the next tile's prefetch
  if constexpr (P::NPASS == 1) {
    if (LD_SMEM) pencil_sync<WARP>();
    pass_st<L, 0>(v, t, st);
  } else {
    if (LD_SMEM) pencil_sync<WARP>();
    pass_st<L, 0>(v, t, sst);
    pencil_sync<WARP>();
    pass_lc<L, SIGN, 1, POW>(v, t, tw, sld);
    if constexpr (P::NPASS == 2) {
      pass_st<L, 1>(v, t, st);
    } else {
      pencil_sync<WARP>();
      pass_st<L, 1>(v, t, sst);
      pencil_sync<WARP>();
      pass_lc<L, SIGN, 2, POW>(v, t, tw, sld);
      pass_st<L, 2>(v, t, st);
    }
  }
}

// ---------------------------------------------------------------- async prefetch (cp.async)
// A thread copies the RMAX pass-0 inputs of its NEXT tile into thread-private shared slots
// (slot s of thread tid at pf[s * nthreads + tid]: conflict-free), so HBM loads stay in
// flight while the current tile is transformed.  src-size 0 zero-fills masked elements.
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
template <int K>   // wait until at most K committed groups are still pending
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory"); }

#ifndef IBK_PFD
#define IBK_PFD 2
#endif
constexpr int PF_DEPTH = IBK_PFD;     // tiles in flight per thread (prefetch depth)

// slot of pass-0 element e for thread t (e = t + q*T + r*NR0  ->  slot q*R0 + r)
template <int L>
__device__ __forceinline__ int pass0_slot(int e, int t) {
  using I = PassI<L, 0>;
  return ((e % I::NR - t) / Plan<L>::T) * I::R + e / I::NR;
}
// call f(slot, e) for the pass-0 elements of thread t
template <int L, class F>
__device__ __forceinline__ void pass0_foreach(int t, F f) {
  using I = PassI<L, 0>;
#pragma unroll
  for (int q = 0; q < I::J; ++q)
#pragma unroll
    for (int r = 0; r < I::R; ++r) f(q * I::R + r, t + q * Plan<L>::T + r * I::NR);
}

}  // namespace ibk
