// xpass_tma.cu — the inverse x pass of step 3 for N1 in [64, 512], persistent and TMA-fed:
//
//   k_xinv_tma : complex-to-real FFT along x of the S1 spectrum -> u^{n+1} (PAPER.md
//                692-695), with the non-finite check of ib_step.
//
// A tile is RB consecutive y rows of one z plane, all 3 components.  A producer warp streams
// tiles into a ring of STAGES shared-memory buffers with cp.async.bulk.tensor (a kx < N/2 row
// box and the Nyquist column box); G consumer groups (own named barrier) take alternate
// tiles.  The tile buffer is reused as the FFT exchange space once a group's pass-0 inputs
// are in registers; results go straight to HBM with coalesced 16-byte stores, so a buffer
// is released as soon as its tile is transformed.  (A TMA-fed forward x pass was measured
// slower than fluid.cu's k_xfwd — its z +- 1 L2 reads need more resident warps than the
// 10-warp, 168-register budget leaves.)
#include <climits>

#include "fft.cuh"
#include "ib_internal.cuh"
#include "tma.cuh"

namespace ibk {

// the x inverse walks the planes top-down: the inverse y pass wrote them bottom-up, so the
// last-written planes are read while still in L2 (138.5 -> 136 us at 256^3)
#ifndef IBK_XI_REV
#define IBK_XI_REV 1
#endif
template <int N>
struct XT {
  static constexpr int M = N / 2;
  static constexpr int T = Plan<M>::T;                  // threads per pencil
  // 2 groups of 3 warps + the producer = 7 warps: the FFT state never spills (spills would
  // miss the small L1 left beside the smem ring).  Measured at 256^3: 2 groups 138 us,
  // 3 groups 142 us, 4 groups 156 us (register-capped), 1 group 160 us.
  static constexpr int RB = 32 / T < N ? 32 / T : N;    // rows per tile
  static constexpr int NTG = 3 * RB * T;                // consumer threads per group
#ifndef IBK_XIG
#define IBK_XIG 2
#endif
  static constexpr int G = IBK_XIG;
  static constexpr int NT = G * NTG;
  static constexpr int NTHR = NT + 32;
  static constexpr int LD = Plan<M>::LD;
  static constexpr size_t PENC = (size_t)3 * RB * LD * 16;          // exchange pencils
  static constexpr int NQ = RB > 8 ? RB : 8;         // Nyquist slot stride (128-B aligned)
  static constexpr size_t XI = (size_t)3 * RB * N * 8 + 3 * NQ * 16; // xinv S1 rows + Nyquist
  static constexpr size_t SI = ((XI > PENC ? XI : PENC) + 1023) & ~(size_t)1023;
#ifndef IBK_XIS
#define IBK_XIS 6
#endif
  static constexpr int SI_STAGES = IBK_XIS;
  // a TMA box is at most 256 doubles wide: rows of N = 512 doubles arrive as HALVES boxes of
  // HC complex each, stored [comp][half][row][HC]
  static constexpr int BOXC = N < 256 ? N : 256;        // doubles per box row
  static constexpr int HALVES = N / BOXC, HC = BOXC / 2;
  static_assert(NTG % 32 == 0, "whole warps per group");
  // each ring stage is always consumed by the same group (see fluid_tma.cu ColCfg)
  static_assert(SI_STAGES % G == 0, "stages per consumer group");
};

// ------------------------------------------------------------------ x inverse (C2R)
// Z'_e = A + i c B, A = X_e + conj X_{M-e}, B = X_e - conj X_{M-e}, c = exp(+2 pi i e/N)
// (see fluid.cu k_xinv), inverse length-M FFT, (r_2k, r_2k+1) pairs straight to HBM.
template <int N>
__global__ void __launch_bounds__(XT<N>::NTHR, 1)
k_xinv_tma(FluidGeom g, const __grid_constant__ CUtensorMap map_main,
           const __grid_constant__ CUtensorMap map_nyq, double *out,
           const double2 *__restrict__ twN, const double2 *__restrict__ twM, long long *flag,
           const long long *dev_n, long long n) {
  using K = XT<N>;
  constexpr int M = K::M, RB = K::RB, T = K::T, LD = K::LD, NTG = K::NTG, G = K::G;
  constexpr int S = K::SI_STAGES;
  const int N2 = g.N2, N3 = g.N3, NYB = N2 / RB;      // N = N1 (row length)
  const int lgy = __ffs(NYB) - 1;                      // NYB is a power of two
  extern __shared__ __align__(1024) double2 smraw[];
  __shared__ uint64_t full[S], done[S];
  __shared__ int bad_any[G];
  double2 *stage0 = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u) / 16u;
  constexpr size_t SW = K::SI / 16;
  const int ntiles = N3 * NYB;
  // output u array: uN3 planes, local plane z at uz0 + z (slab: ghost planes around)
  const size_t Vu = (size_t)N * N2 * g.uN3;
  const int uz0 = g.uz0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&done[s], 1); }
    fence_mbar_init();
  }
  if (threadIdx.x < G) bad_any[threadIdx.x] = 0;
  // C2R pre-twiddles staged once per CTA (persistent): shared loads in the pass-0 gather
  // instead of L1 hits on the table
  __shared__ double2 twx[M];
  for (int e = threadIdx.x; e < M; e += blockDim.x) twx[e] = twN[e];
  __syncthreads();

  if (threadIdx.x >= K::NT) {                             // -------------- producer warp
    if (threadIdx.x == K::NT) {
      prefetch_tmap(&map_main);
      prefetch_tmap(&map_nyq);
      int i = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
        const int s = i % S;
        if (i >= S) mbar_wait(&done[s], ((i / S) - 1) & 1);
        const int z = IBK_XI_REV ? N3 - 1 - (tile >> lgy) : (tile >> lgy), y0 = (tile & (NYB - 1)) * RB;
        double2 *b = stage0 + (size_t)s * SW;            // [3][RB][M] then [3][RB] Nyquist
        mbar_expect_tx(&full[s], (uint32_t)(3 * RB * (M + 1) * 16));
        for (int c = 0; c < 3; ++c) {
          const int r0 = (c * N3 + z) * N2 + y0;
          for (int hf = 0; hf < K::HALVES; ++hf)
            tma_load_2d(b + ((size_t)c * K::HALVES + hf) * RB * K::HC, &map_main, hf * K::BOXC, r0,
                        &full[s]);
          tma_load_2d(b + (size_t)3 * RB * M + c * K::NQ, &map_nyq, 2 * M, r0, &full[s]);
        }
      }
    }
    return;
  }

  const int grp = threadIdx.x / NTG, gtid = threadIdx.x % NTG, bar = 1 + grp;
  const int t = gtid % T, pencil = gtid / T, row = pencil % RB, comp = pencil / RB;
  const long long step = dev_n ? *dev_n : n;
  int i = grp;
  bool bad = false;
  for (int tile = blockIdx.x + grp * gridDim.x; tile < ntiles; tile += G * gridDim.x, i += G) {
    const int s = i % S;
    if (s % G != grp) __trap();                          // ring-ownership rule (XT)
    const int z = IBK_XI_REV ? N3 - 1 - (tile >> lgy) : (tile >> lgy), y0 = (tile & (NYB - 1)) * RB;
    double2 *sm = stage0 + (size_t)s * SW;
    // X_e of this row: half e / HC, position e % HC (one half when N <= 256)
    const double2 *in = sm + (size_t)comp * RB * M + (size_t)row * K::HC;
    auto X_at = [&](int e) -> double2 {
      return in[(e / K::HC) * RB * K::HC + (e % K::HC)];
    };
    mbar_wait(&full[s], (i / S) & 1);
    const double2 nyq = sm[(size_t)3 * RB * M + comp * K::NQ + row];
    double2 *o2 = reinterpret_cast<double2 *>(out + comp * Vu + ((size_t)(uz0 + z) * N2 + (y0 + row)) * N);
    auto ld = [&](int e) -> double2 {
      double2 Xk = X_at(e), Xm = e == 0 ? nyq : X_at(M - e);
      if (e == 0) { Xk.y = 0.0; Xm.y = 0.0; }      // X_0, X_{N/2} are real
      const double2 A = make_double2(Xk.x + Xm.x, Xk.y - Xm.y);
      const double2 B = make_double2(Xk.x - Xm.x, Xk.y + Xm.y);
      const double2 cB = cmul(cconj(twx[e]), B);
      return make_double2(A.x - cB.y, A.y + cB.x);
    };
    auto st = [&](int k, double2 v) {
      bad |= !(isfinite(v.x) && isfinite(v.y));
      o2[k] = v;
    };
    // pass-0 loads read the stage (all group threads) before any pencil store aliases it
    auto sync_after_load = [&]() { named_bar(bar, NTG); };
    double2 *sp = sm + pencil * LD;
    // power twiddles at N1 = 512 only (measured: 1084 -> 991 us there, +8 us at 256)
    fft_io<M, +1, false, true, (N >= 512)>(sp, t, twM, ld, st, sync_after_load);
    // the pencil stores above are generic-proxy writes into the stage the producer refills
    // with TMA (async proxy): order them before the release
    fence_proxy_async();
    named_bar(bar, NTG);
    if (gtid == 0) mbar_arrive(&done[s]);
  }
  if (flag && bad) bad_any[grp] = 1;
  named_bar(1 + grp, NTG);
  if (flag && gtid == 0 && bad_any[grp]) atomicMin(flag, step);
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn_x() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// rows x cols doubles (row pitch `pitch` bytes), box box_cols x box_rows, no swizzle
static bool encode_rows(CUtensorMap *m, const void *base, uint64_t rows, uint64_t cols,
                        uint64_t pitch, uint32_t box_cols, uint32_t box_rows) {
  auto fn = encode_fn_x();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows}, strides[1] = {pitch};
  cuuint32_t box[2] = {box_cols, box_rows}, es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void *>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int xt_rb(int N) {
  switch (N) {
    case 64: return XT<64>::RB;
    case 128: return XT<128>::RB;
    case 256: return XT<256>::RB;
    case 512: return XT<512>::RB;
    default: return 0;
  }
}

bool xpass_supported(int N) { return N >= 64 && N <= 512; }   // N = N1

bool xpass_encode_s1(const FluidGeom &g, const double2 *spec, XMapsS *m) {
  const int N = g.N1;
  if (!xpass_supported(N) || g.N2 % xt_rb(N)) return false;
  const uint64_t rows = (uint64_t)3 * g.N2 * g.N3;
  const uint32_t boxc = N < 256 ? N : 256;
  return encode_rows(&m->main, spec, rows, 2 * (g.M + 1), (uint64_t)g.P * 16, boxc, xt_rb(N)) &&
         encode_rows(&m->nyq, spec, rows, 2 * (g.M + 1), (uint64_t)g.P * 16, 2, xt_rb(N));
}

template <class Kern>
static int grid_for(Kern k, int threads, size_t smem, int ntiles) {
  int per = 0;
  const int nsm = sm_count();
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, threads, smem);
  if (per < 1) per = 1;
  return ntiles < per * nsm ? ntiles : per * nsm;
}

template <int N>
static cudaError_t xinv_n(const FluidGeom &g, const XMapsS &m, double *out, const double2 *twN,
                          const double2 *twM, long long *flag, const long long *dev_n,
                          long long n, cudaStream_t s) {
  using K = XT<N>;
  const size_t smem = (size_t)K::SI_STAGES * K::SI + 1024;
  static PerDeviceOnce attr;
  const int dev = current_device();
  if (!attr.done(dev)) {
    cudaError_t e = cudaFuncSetAttribute(k_xinv_tma<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr.mark(dev);
  }
  const int grid = grid_for(k_xinv_tma<N>, K::NTHR, smem, g.N3 * (g.N2 / K::RB));
  k_xinv_tma<N><<<grid, K::NTHR, smem, s>>>(g, m.main, m.nyq, out, twN, twM, flag, dev_n, n);
  return cudaGetLastError();
}

cudaError_t launch_xinv_tma(const FluidGeom &g, const XMapsS &m, double *out,
                            const double2 *twN, const double2 *twM, long long *flag,
                            const long long *dev_n, long long n, cudaStream_t s) {
  switch (g.N1) {
    case 64: return xinv_n<64>(g, m, out, twN, twM, flag, dev_n, n, s);
    case 128: return xinv_n<128>(g, m, out, twN, twM, flag, dev_n, n, s);
    case 256: return xinv_n<256>(g, m, out, twN, twM, flag, dev_n, n, s);
    case 512: return xinv_n<512>(g, m, out, twN, twM, flag, dev_n, n, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ibk
