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
#include "tma.cuh"

namespace ibk {

// ------------------------------------------------------------------ tile configuration
#ifndef IBK_XRB
#define IBK_XRB 32   // rows x threads-per-pencil: RB = 4 rows at N1 = 256 (5 CTAs per SM)
#endif
#ifndef IBK_XRB512
#define IBK_XRB512 32   // the same product at N1 = 512: RB = 2 rows
#endif
template <int N> struct XCfg {      // x passes: RB rows of one z-plane per CTA
  static constexpr int M = N / 2;
  static constexpr int T = Plan<M>::T;
  static constexpr int RBT = N >= 512 ? IBK_XRB512 : IBK_XRB;
  static constexpr int RB = (RBT / T) < N ? (RBT / T) : N;
};
#ifndef IBK_YC
#define IBK_YC 8
#endif
template <int N> struct YCfg {      // y pass: C consecutive kx columns per CTA (256-byte rows
  static constexpr int T = Plan<N>::T;   // on the large-pitch side, see tools/membench.cu)
  static constexpr int C = IBK_YC;
};
#ifndef IBK_ZC
#define IBK_ZC 2
#endif
#ifndef IBK_ZMINB
#define IBK_ZMINB 4
#endif
template <int N> struct ZCfg {      // z pass: C consecutive kx columns x 3 components per CTA
  static constexpr int T = Plan<N>::T;
  static constexpr int C0 = (16 * IBK_ZC) / T;
  static constexpr int C = C0 < 1 ? 1 : (C0 > 32 ? 32 : C0);
  static constexpr int MINB = IBK_ZMINB;                    // CTAs/SM the registers must allow
};

__device__ __forceinline__ long long step_of(const long long *dev_n, long long n) {
  return dev_n ? *dev_n : n;
}

// ------------------------------------------------------------------ tables
// Per-axis tables of a lattice axis of length N: twiddles exp(-2 pi i t/N), the D0 symbol
// s and -symbol of D+D- l; twM (x axis only, may be null): exp(-2 pi i t/M), M = N/2.
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
  if (twM && t < M) {
    double sn, cs;
    sincospi(2.0 * (double)t / (double)M, &sn, &cs);
    twM[t] = make_double2(cs, -sn);
  }
}

cudaError_t init_axis_table(double2 *twN, int N, double *s, double *l, double h, cudaStream_t st) {
  k_init_tables<<<(N + 127) / 128, 128, 0, st>>>(twN, N, nullptr, 0, s, l, h);
  return cudaGetLastError();
}

cudaError_t init_tables(ib_ctx *c) {
  const int L[3] = {c->g.N1, c->g.N2, c->g.N3};
  for (int a = 0; a < 3; ++a) {
    k_init_tables<<<(L[a] + 127) / 128, 128, 0, c->stream>>>(
        c->tw[a], L[a], a == 0 ? c->twM : nullptr, L[0] / 2, c->sym_s[a], c->sym_l[a], c->g.h);
    c->launches++;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ x forward
// MODE 0: step (r from u, F; F re-zeroed; R2C-x); 1: r only -> r_out; 2: R2C-x of `in`.
// Thread (pencil = comp*RB + row, t): t fastest, so a warp's accesses along x are
// contiguous.  The CTA first copies rows y0-1 .. y0+RB of plane z (3 components) to
// shared memory with cp.async; each thread then computes r at the 2*RMAX cells of its
// first-pass elements (z_e = r_2e + i r_2e+1) from that tile plus the z +- 1 rows (L2),
// straight into registers.  The tile is then reused as the FFT exchange buffer.
// CTAs per SM the registers must allow: 5 (15 warps, <= 128 registers) at N1 <= 256 (266
// vs 287 us at 256^3 with 4; 6 spill); 4 at N1 = 512, whose 48 KB tiles fit only 4 per SM
// anyway (2407 vs 2620 us at 512^3 with the 128-register cap)
#ifndef IBK_XMINB
#define IBK_XMINB (N >= 512 ? (XCfg<N>::RB >= 4 ? 3 : 4) : 5)
#endif
template <int N, int MODE>
__global__ void __launch_bounds__(3 * XCfg<N>::RB * XCfg<N>::T, IBK_XMINB)
k_xfwd(FluidGeom g, const double *__restrict__ u, double *F, unsigned *rowflag,
       const double *__restrict__ in, double *r_out, double2 *spec,
       const double2 *__restrict__ twN, const double2 *__restrict__ twM,
       const __grid_constant__ CUtensorMap map_rows, const __grid_constant__ CUtensorMap map_row1,
       int use_tma) {
  constexpr int M = N / 2, RB = XCfg<N>::RB, T = XCfg<N>::T, LD = Plan<M>::LD;
  constexpr int NC = MODE == 2 ? 1 : 3, UR = RB + 2;
  extern __shared__ __align__(128) double2 smraw_x[];
  __shared__ uint64_t tbar;
  // 128-byte aligned tile (TMA destination); offset arithmetic keeps accesses LDS/STS
  double2 *sm = smraw_x + ((128u - (smem_u32(smraw_x) & 127u)) & 127u) / 16u;
  double *ut = reinterpret_cast<double *>(sm);     // u tile [comp][UR][N1]
  const int N2 = g.N2, N3 = g.N3;                  // rows per plane, planes
  const int z = blockIdx.y, y0 = blockIdx.x * RB;
  // u array: uN3 planes, local plane z at uz0 + z (slab: ghost planes around the owned ones)
  const int uN3 = g.uN3, zu = g.uz0 + z;
  const size_t Vu = (size_t)N * N2 * uN3;
  const int t = threadIdx.x % T, pencil = threadIdx.x / T;
  const int row = pencil % RB, comp = pencil / RB, y = y0 + row;
  const size_t V = (size_t)g.V;
  const size_t rowbase = ((size_t)z * N2 + y) * N;
  const double cu = g.rho / g.dt, ra = g.rho * g.invh;
  // F is only read on rows the spread touched (row flags), else taken as 0; the flag is
  // loaded before the tile wait so that its latency overlaps the TMA transfer
  const unsigned rflag = (MODE == 0 && rowflag) ? rowflag[(size_t)z * N2 + y] : 1u;
  // z -+ 1: periodic on the whole lattice; in a slab the neighbours are ghost planes
  const int zmi = g.slab ? zu - 1 : ((z + N3 - 1) & (N3 - 1));
  const int zpi = g.slab ? zu + 1 : ((z + 1) & (N3 - 1));
  const size_t zm = ((size_t)zmi * N2 + y) * N;
  const size_t zp = ((size_t)zpi * N2 + y) * N;
  const double *uc_ = u + (MODE == 2 ? 0 : comp * Vu);
  // the z -+ 1 rows (L2) of the first ZPF pass-0 slots are requested before the tile wait,
  // so that their latency overlaps the TMA transfer instead of stalling the stencil
#ifndef IBK_XZPF
#define IBK_XZPF 2
#endif
  constexpr int ZPF = MODE == 2 ? 0 : IBK_XZPF;
  double2 zpre[ZPF > 0 ? 2 * ZPF : 1] = {};
  if constexpr (ZPF > 0) {
    pass0_foreach<M>(t, [&](int slot, int e) {
      if (slot < ZPF) {
        zpre[2 * slot] = __ldg(reinterpret_cast<const double2 *>(uc_ + zm + 2 * e));
        zpre[2 * slot + 1] = __ldg(reinterpret_cast<const double2 *>(uc_ + zp + 2 * e));
      }
    });
  }
  // N1 = 512: the z -+ 1 rows of the remaining slots are prefetched into L1 (no registers),
  // also before the tile wait: x forward 2244 -> 2093 us at 512^3 (6 slots: 2192); at
  // N1 = 256 the same prefetch is neutral to slower (243.7 -> 245.9 us, 6 slots 250), so off
#ifndef IBK_XL1PF
#define IBK_XL1PF (N >= 512 ? 16 : 0)
#endif
  constexpr int L1PF = IBK_XL1PF;
  if constexpr (MODE != 2 && L1PF > 0) {
    pass0_foreach<M>(t, [&](int slot, int e) {
      if (slot >= ZPF && slot < ZPF + L1PF) {
        asm volatile("prefetch.global.L1 [%0];" ::"l"(uc_ + zm + 2 * e));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(uc_ + zp + 2 * e));
      }
    });
  }
  // the F of a flagged row is prefetched into L1 likewise (x forward 2089 -> 2039 us at 512^3,
  // 243.7 -> 242.2 us at 256^3)
#ifndef IBK_XFPF
#define IBK_XFPF 1
#endif
  if constexpr (MODE == 0 && IBK_XFPF) {
    if (rflag != 0)
      pass0_foreach<M>(t, [&](int slot, int e) {
        asm volatile("prefetch.global.L1 [%0];" ::"l"(F + comp * V + rowbase + 2 * e));
      });
  }
  if (MODE != 2 && use_tma) {   // one thread streams the 3 x (RB + 2) rows with TMA
    if (threadIdx.x == 0) {
      mbar_init(&tbar, 1);
      fence_mbar_init();
      mbar_expect_tx(&tbar, (uint32_t)(3 * UR * N * 8));
      for (int c = 0; c < 3; ++c) {
        const int rb = (c * uN3 + zu) * N2;
        if constexpr (N > 256) {   // rows of 512 doubles: 3-D view (256, 2 halves, row)
          tma_load_3d(ut + ((size_t)c * UR + 1) * N, &map_rows, 0, 0, rb + y0, &tbar);
          tma_load_3d(ut + (size_t)c * UR * N, &map_row1, 0, 0, rb + ((y0 - 1 + N2) & (N2 - 1)), &tbar);
          tma_load_3d(ut + ((size_t)c * UR + RB + 1) * N, &map_row1, 0, 0, rb + ((y0 + RB) & (N2 - 1)), &tbar);
        } else {
          tma_load_2d(ut + ((size_t)c * UR + 1) * N, &map_rows, 0, rb + y0, &tbar);
          tma_load_2d(ut + (size_t)c * UR * N, &map_row1, 0, rb + ((y0 - 1 + N2) & (N2 - 1)), &tbar);
          tma_load_2d(ut + ((size_t)c * UR + RB + 1) * N, &map_row1, 0, rb + ((y0 + RB) & (N2 - 1)), &tbar);
        }
      }
    }
    __syncthreads();                                // barrier initialised before anyone waits
    mbar_wait(&tbar, 0);
  } else if (MODE != 2) {
    constexpr int CH = N / 2;                      // 16-byte chunks per row
    for (int idx = threadIdx.x; idx < 3 * UR * CH; idx += blockDim.x) {
      const int ch = idx % CH, rr = (idx / CH) % UR, cc = idx / (CH * UR);
      const int yy = (y0 - 1 + rr + N2) & (N2 - 1);
      cp_async16(ut + ((size_t)cc * UR + rr) * N + 2 * ch,
                 u + cc * Vu + ((size_t)zu * N2 + yy) * N + 2 * ch, true);
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
  }
  const bool hasF = MODE == 1 || (MODE == 0 && rflag != 0);
  const double *own = ut + ((size_t)comp * UR + row + 1) * N;        // this row, own comp

  // r at the cell pair (2e, 2e+1) of this thread's component: sum_k u_k D_k^{+-} u_i
  // with the backward difference for u_k > 0 (and u_k = 0, Z5), the forward one for
  // u_k < 0 (PAPER.md 676-691); all operands loaded unconditionally.
  auto rhs2 = [&](int e, int slot) -> double2 {
    const int x = 2 * e;
    const double2 v0 = *reinterpret_cast<const double2 *>(ut + (0 * UR + row + 1) * N + x);
    const double2 v1 = *reinterpret_cast<const double2 *>(ut + (1 * UR + row + 1) * N + x);
    const double2 v2 = *reinterpret_cast<const double2 *>(ut + (2 * UR + row + 1) * N + x);
    const double2 c = comp == 0 ? v0 : (comp == 1 ? v1 : v2);
    const double xm = own[(x + N - 1) & (N - 1)];
    const double xp = own[(x + 2) & (N - 1)];
    const double2 a_ym = *reinterpret_cast<const double2 *>(own - N + x);
    const double2 a_yp = *reinterpret_cast<const double2 *>(own + N + x);
    const double2 a_zm = slot < ZPF ? zpre[2 * slot]
                                    : __ldg(reinterpret_cast<const double2 *>(uc_ + zm + x));
    const double2 a_zp = slot < ZPF ? zpre[2 * slot + 1]
                                    : __ldg(reinterpret_cast<const double2 *>(uc_ + zp + x));
    double2 Fi = make_double2(0.0, 0.0);
    double2 *Fp = reinterpret_cast<double2 *>(F + comp * V + rowbase + x);
    if (hasF) Fi = *Fp;
    const double dx0 = v0.x < 0.0 ? c.y - c.x : c.x - xm;
    const double dx1 = v0.y < 0.0 ? xp - c.y : c.y - c.x;
    const double dy0 = v1.x < 0.0 ? a_yp.x - c.x : c.x - a_ym.x;
    const double dy1 = v1.y < 0.0 ? a_yp.y - c.y : c.y - a_ym.y;
    const double dz0 = v2.x < 0.0 ? a_zp.x - c.x : c.x - a_zm.x;
    const double dz1 = v2.y < 0.0 ? a_zp.y - c.y : c.y - a_zm.y;
    const double adv0 = v0.x * dx0 + v1.x * dy0 + v2.x * dz0;
    const double adv1 = v0.y * dx1 + v1.y * dy1 + v2.y * dz1;
    if (MODE == 0 && hasF && (Fi.x != 0.0 || Fi.y != 0.0)) *Fp = make_double2(0.0, 0.0);
    return make_double2(cu * c.x - ra * adv0 + Fi.x, cu * c.y - ra * adv1 + Fi.y);
  };

  double2 rr[Plan<M>::RMAX];
  pass0_foreach<M>(t, [&](int slot, int e) {
    rr[slot] = MODE == 2 ? __ldg(reinterpret_cast<const double2 *>(in + rowbase) + e) : rhs2(e, slot);
  });
  if (MODE == 1) {      // r only (debug)
    pass0_foreach<M>(t, [&](int slot, int e) {
      reinterpret_cast<double2 *>(r_out + comp * V + rowbase)[e] = rr[slot];
    });
    return;
  }
  auto ld = [&](int e, int slot) { return rr[slot]; };
  double2 *sp = sm + pencil * LD;
  // the last pass stores unswizzled (consecutive e per quarter-warp): the split below then
  // reads both k and M - k runs without bank conflicts
  auto sst = [sp](int e, double2 v) { sp[e] = v; };
  auto bar = []() { __syncthreads(); };             // u tile dead before pencils alias it
  fft_io<M, -1, false, true, true>(sp, t, twM, ld, sst, bar);   // power twiddles (measured)
  __syncthreads();
  if (MODE == 0 && rowflag && threadIdx.x < RB) rowflag[(size_t)z * N2 + y0 + threadIdx.x] = 0u;
  // split the length-M transform Z of z_n = r_2n + i r_2n+1 into X_k, k = 0..M:
  // E = (Z_k + conj Z_{M-k})/2, O = -i (Z_k - conj Z_{M-k})/2, X_k = E + w^k O,
  // X_{M-k} = conj(E - w^k O), w = exp(-2 pi i/N).
  constexpr int H = M / 2 + 1;
  for (int idx = threadIdx.x; idx < NC * RB * H; idx += blockDim.x) {
    const int pc = idx / H, k = idx % H;
    const int cp = pc / RB, rw = pc % RB;
    const double2 Zk = sm[pc * LD + k];
    const double2 Zm = sm[pc * LD + ((M - k) & (M - 1))];
    const double2 E = make_double2(0.5 * (Zk.x + Zm.x), 0.5 * (Zk.y - Zm.y));
    const double2 O = make_double2(0.5 * (Zk.y + Zm.y), -0.5 * (Zk.x - Zm.x));
    const double2 wO = cmul(__ldg(&twN[k]), O);
    double2 *out = spec + (((size_t)cp * N3 + z) * N2 + (y0 + rw)) * g.P;
    out[k] = cadd(E, wO);
    if (k != M - k) out[M - k] = cconj(csub(E, wO));
  }
}

template <int N>
static cudaError_t launch_xfwd_n(const FluidGeom &g, int mode, const double *u, double *F,
                                 unsigned *rowflag, const double *in, double *r_out,
                                 double2 *spec, const double2 *twN, const double2 *twM,
                                 const XMapsU *um, cudaStream_t s) {
  using X = XCfg<N>;
  if (g.N2 % X::RB) return cudaErrorInvalidValue;     // ib_create3 checks this
  dim3 grid(g.N2 / X::RB, g.N3);
  const int nc = mode == 2 ? 1 : 3;
  const size_t fft = (size_t)nc * X::RB * Plan<N / 2>::LD * sizeof(double2);
  const size_t tile = mode == 2 ? 0 : (size_t)3 * (X::RB + 2) * N * sizeof(double);
  const size_t smem = (fft > tile ? fft : tile) + 128;
  const int threads = nc * X::RB * X::T;
  // TMA row boxes (N <= 256 doubles per box) when the caller encoded maps of u
  CUtensorMap rows{}, row1{};
  const int use_tma = (mode != 2 && um && um->ok) ? 1 : 0;
  if (use_tma) { rows = um->rows; row1 = um->row1; }
  if (mode == 0)
    k_xfwd<N, 0><<<grid, threads, smem, s>>>(g, u, F, rowflag, in, r_out, spec, twN, twM, rows, row1, use_tma);
  else if (mode == 1)
    k_xfwd<N, 1><<<grid, threads, smem, s>>>(g, u, F, nullptr, in, r_out, spec, twN, twM, rows, row1, use_tma);
  else
    k_xfwd<N, 2><<<grid, threads, smem, s>>>(g, u, F, nullptr, in, r_out, spec, twN, twM, rows, row1, 0);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ y pass
// Spectrum layouts (complex elements, row pitch P):
//   S1 [comp][z][y][kx]  (x passes):   z stride N*P, y stride P
//   S2 [comp][ky][z][kx] (z pass):     z stride P,   ky stride N*P
// The forward y pass reads S1 and writes S2, the inverse reads S2 and writes S1, so the
// z pass streams contiguous (ky, comp) slabs; the y passes take the large-pitch side with
// 256-byte row segments (C = 16 columns), which tools/membench.cu measured at ~6.5 TB/s.
// Persistent CTAs walk the (kx-block, z, comp) tiles; thread (col, t), col fastest.  Each
// thread cp.async-prefetches the pass-0 inputs of its next tile into private smem slots
// right after loading the current ones, so HBM loads overlap the transform.
template <int N, int SIGN>
__global__ void __launch_bounds__(YCfg<N>::C * YCfg<N>::T)
k_ypass(FluidGeom g, const double2 *in, double2 *out, size_t in_zs, size_t in_es,
        size_t out_zs, size_t out_es, int ncomp, const double2 *__restrict__ twN) {
  constexpr int C = YCfg<N>::C, LD = Plan<N>::LD, NT = C * Plan<N>::T;
  const int M = g.M, N3 = g.N3;                     // kx in [0, M]; z planes
  extern __shared__ double2 sm[];
  double2 *pf = sm + C * LD;              // prefetch slots [PF_DEPTH][RMAX][NT]
  constexpr int SLOTS = Plan<N>::RMAX * NT;
  const int col = threadIdx.x % C, t = threadIdx.x / C;
  const int NBLK = (M + 1 + C - 1) / C;
  const int ntiles = NBLK * N3 * ncomp;
  const size_t cstride = (size_t)N * N3 * g.P;
  auto prefetch = [&](int tile, int stage) {
    if (tile < ntiles) {
      const int kx = (tile % NBLK) * C + col, z = (tile / NBLK) % N3, comp = tile / (NBLK * N3);
      const bool ok = kx <= M;
      const double2 *ib = in + comp * cstride + z * in_zs + (ok ? kx : 0);
      double2 *dst = pf + stage * SLOTS + threadIdx.x;
      pass0_foreach<N>(t, [&](int slot, int e) { cp_async16(dst + slot * NT, ib + e * in_es, ok); });
    }
    cp_async_commit();                   // (possibly empty) group per tile keeps the count
  };
#pragma unroll
  for (int d = 0; d < PF_DEPTH; ++d) prefetch(blockIdx.x + d * gridDim.x, d);
  int stage = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int kx = (tile % NBLK) * C + col, z = (tile / NBLK) % N3, comp = tile / (NBLK * N3);
    const bool ok = kx <= M;
    double2 *ob = out + comp * cstride + z * out_zs + kx;
    cp_async_wait<PF_DEPTH - 1>();
    const double2 *src = pf + stage * SLOTS + threadIdx.x;
    auto ld = [&](int e, int slot) { return src[slot * NT]; };
    auto st = [&](int e, double2 v) { if (ok) ob[e * out_es] = v; };
    auto nxt = [&]() { prefetch(tile + PF_DEPTH * gridDim.x, stage); };
    fft_io<N, SIGN, false, false>(sm + col * LD, t, twN, ld, st, nxt);
    stage = stage + 1 == PF_DEPTH ? 0 : stage + 1;
    __syncthreads();                               // exchange pencils reused by next tile
  }
}

template <class K>
static int persistent_grid(K kernel, int threads, size_t smem, int ntiles) {
  const int nsm = sm_count();
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem);
  if (per < 1) per = 1;
  return ntiles < per * nsm ? ntiles : per * nsm;
}

template <int N>
static cudaError_t launch_ypass_n(const FluidGeom &g, int sign, const double2 *in, int in_layout,
                                  double2 *out, int out_layout, int ncomp, const double2 *twN,
                                  cudaStream_t s) {
  using Y = YCfg<N>;
  const int threads = Y::C * Y::T;
  const size_t smem = ((size_t)Y::C * Plan<N>::LD + (size_t)PF_DEPTH * Plan<N>::RMAX * threads) * sizeof(double2);
  const int ntiles = ((g.M + 1 + Y::C - 1) / Y::C) * g.N3 * ncomp;
  // S1 [comp][z][y][kx]: z stride N2 P, y stride P; S2 [comp][ky][z][kx]: z stride P,
  // ky stride N3 P  (N = N2 here)
  const size_t P = g.P, N2P = (size_t)N * g.P, N3P = (size_t)g.N3 * g.P;
  const size_t izs = in_layout == 1 ? N2P : P, ies = in_layout == 1 ? P : N3P;
  const size_t ozs = out_layout == 1 ? N2P : P, oes = out_layout == 1 ? P : N3P;
  if (sign < 0) {
    const int grid = persistent_grid(k_ypass<N, -1>, threads, smem, ntiles);
    k_ypass<N, -1><<<grid, threads, smem, s>>>(g, in, out, izs, ies, ozs, oes, ncomp, twN);
  } else {
    const int grid = persistent_grid(k_ypass<N, +1>, threads, smem, ntiles);
    k_ypass<N, +1><<<grid, threads, smem, s>>>(g, in, out, izs, ies, ozs, oes, ncomp, twN);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ z pass + solve
// Per mode k (DESIGN.md §2 S3c):  d = rho/dt + mu (l(kx) + l(ky) + l(kz)),
//   u^ = (r^ - s (s.r^)/|s|^2) / (d N^3),   p^ = -i (s.r^)/|s|^2 / N^3,
//   and on the 8 null modes (every k_a in {0, N/2}): u^ = r^/(d N^3), p^ = 0.
// Thread (t, col, group), t fastest (a quarter-warp is 8 jobs of one pencil, which the
// PAD swizzle keeps conflict-free); groups 0..2 = velocity components, 3 = pressure.
// Forward FFT: HBM -> registers -> smem exchange -> natural-order modes in smem; solve
// in smem; inverse FFT: smem -> registers -> smem exchange -> HBM.
template <int N, int MODE, bool PRESS>
__global__ void __launch_bounds__((PRESS ? 4 : 3) * ZCfg<N>::C * ZCfg<N>::T, PRESS ? 1 : ZCfg<N>::MINB)
k_zpass(FluidGeom g, double2 *spec, double2 *pspec, const double2 *__restrict__ twN, Sym sym) {
  constexpr int C = ZCfg<N>::C, T = ZCfg<N>::T, LD = Plan<N>::LD;
  constexpr int NG = PRESS ? 4 : 3, NT = NG * C * T;
  const int M = g.M, N2 = g.N2;                     // kx in [0, M]; ky in [0, N2)
  const int NBLK = (M + 1 + C - 1) / C;
  extern __shared__ double2 sm[];
  double2 *pf = sm + NG * C * LD;         // prefetch slots [PF_DEPTH][RMAX][NT]
  constexpr int SLOTS = Plan<N>::RMAX * NT;
  const int t = threadIdx.x % T, col = (threadIdx.x / T) % C, grp = threadIdx.x / (C * T);
  const int ntiles = NBLK * N2;
  const size_t zs = g.P;                           // S2 layout: [comp][ky][z][kx]
  double2 *sp = sm + (grp * C + col) * LD;
  auto prefetch = [&](int tile, int stage) {
    if (tile < ntiles) {
      const int kx = (tile % NBLK) * C + col, ky = tile / NBLK;
      const bool ok = kx <= M && grp < 3;
      const double2 *b = spec + ((size_t)(grp < 3 ? grp : 0) * N2 + ky) * N * g.P + (ok ? kx : 0);
      double2 *dst = pf + stage * SLOTS + threadIdx.x;
      pass0_foreach<N>(t, [&](int slot, int e) { cp_async16(dst + slot * NT, b + e * zs, ok); });
    }
    cp_async_commit();
  };
#pragma unroll
  for (int d = 0; d < PF_DEPTH; ++d) prefetch(blockIdx.x + d * gridDim.x, d);
  int stage = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int col0 = (tile % NBLK) * C, ky = tile / NBLK, kx = col0 + col;
    const bool ok = kx <= M;
    double2 *base = grp < 3 ? spec + ((size_t)grp * N2 + ky) * N * g.P + kx
                            : pspec + (size_t)ky * N * g.P + kx;
    auto gst = [&](int e, double2 v) { if (ok) base[e * zs] = v; };
    auto sst = [sp](int e, double2 v) { sp[PAD(e)] = v; };
    auto sld = [sp](int e) { return sp[PAD(e)]; };
    cp_async_wait<PF_DEPTH - 1>();
    const int cur = stage;
    stage = stage + 1 == PF_DEPTH ? 0 : stage + 1;
    const double2 *src = pf + cur * SLOTS + threadIdx.x;
    auto ld = [&](int e, int slot) { return src[slot * NT]; };
    auto nxt = [&]() { prefetch(tile + PF_DEPTH * gridDim.x, cur); };
    if (MODE == 1) {     // forward only (debug entry point)
      fft_io<N, -1, false, true>(sp, t, twN, ld, gst, nxt);
      __syncwarp();
      continue;
    }
    fft_io<N, -1, false, true>(sp, t, twN, ld, sst, nxt);
    __syncthreads();
    {
      const double sy = sym.sy[ky], ly = sym.ly[ky];
      const bool ny = (ky == 0) || (2 * ky == N2);
      const double invV = 1.0 / (double)g.V;
      for (int idx = threadIdx.x; idx < C * N; idx += blockDim.x) {
        const int c = idx / N, kz = idx % N, kxx = col0 + c;
        if (kxx > M) continue;
        const double sx = sym.sx[kxx], sz = sym.sz[kz];
        const double d = g.rho / g.dt + g.mu * (sym.lx[kxx] + ly + sym.lz[kz]);
        double2 *q0 = sm + (0 * C + c) * LD + PAD(kz);
        double2 *q1 = q0 + C * LD;
        double2 *q2 = q1 + C * LD;
        const double2 r0 = *q0, r1 = *q1, r2 = *q2;
        const bool nul = ny && (kxx == 0 || kxx == M) && (kz == 0 || 2 * kz == N);
        if (nul) {
          const double inv = invV / d;
          *q0 = cscale(r0, inv); *q1 = cscale(r1, inv); *q2 = cscale(r2, inv);
          if (PRESS) q2[C * LD] = make_double2(0.0, 0.0);
        } else {
          // one division: w = 1/(d |s|^2) gives 1/d = w |s|^2 and 1/|s|^2 = w d
          const double s2 = sx * sx + sy * sy + sz * sz;
          const double w = 1.0 / (d * s2);
          const double is2 = w * d, inv = invV * (w * s2);
          const double2 q = make_double2((sx * r0.x + sy * r1.x + sz * r2.x) * is2,
                                         (sx * r0.y + sy * r1.y + sz * r2.y) * is2);
          *q0 = make_double2((r0.x - sx * q.x) * inv, (r0.y - sx * q.y) * inv);
          *q1 = make_double2((r1.x - sy * q.x) * inv, (r1.y - sy * q.y) * inv);
          *q2 = make_double2((r2.x - sz * q.x) * inv, (r2.y - sz * q.y) * inv);
          if (PRESS) q2[C * LD] = make_double2(q.y * invV, -q.x * invV);
        }
      }
    }
    __syncthreads();
    fft_io<N, +1, true, true>(sp, t, twN, sld, gst);
    __syncwarp();                                  // pencil reused by the next tile
  }
}

template <int N>
static cudaError_t launch_zpass_n(const FluidGeom &g, int mode, double2 *spec, double2 *pspec,
                                  const double2 *twN, const Sym &sym, cudaStream_t s) {
  using Z = ZCfg<N>;
  const int ntiles = ((g.M + 1 + Z::C - 1) / Z::C) * g.N2;
  const int t3 = 3 * Z::C * Z::T, t4 = 4 * Z::C * Z::T;
  const size_t smem3 = ((size_t)3 * Z::C * Plan<N>::LD + (size_t)PF_DEPTH * Plan<N>::RMAX * t3) * sizeof(double2);
  const size_t smem4 = ((size_t)4 * Z::C * Plan<N>::LD + (size_t)PF_DEPTH * Plan<N>::RMAX * t4) * sizeof(double2);
  if (mode == 1) {
    const int grid = persistent_grid(k_zpass<N, 1, false>, t3, smem3, ntiles);
    k_zpass<N, 1, false><<<grid, t3, smem3, s>>>(g, spec, pspec, twN, sym);
  } else if (pspec) {
    const int grid = persistent_grid(k_zpass<N, 0, true>, t4, smem4, ntiles);
    k_zpass<N, 0, true><<<grid, t4, smem4, s>>>(g, spec, pspec, twN, sym);
  } else {
    const int grid = persistent_grid(k_zpass<N, 0, false>, t3, smem3, ntiles);
    k_zpass<N, 0, false><<<grid, t3, smem3, s>>>(g, spec, pspec, twN, sym);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ x inverse (C2R)
// Z'_e = A + i c B with A = X_e + conj X_{M-e}, B = X_e - conj X_{M-e}, c = exp(+2 pi i e/N)
// is formed while loading (both X read from HBM/L1); the inverse length-M FFT of Z' is
// N (r_even + i r_odd), written straight from the last pass as (r_2k, r_2k+1) pairs.
template <int N>
__global__ void __launch_bounds__(3 * XCfg<N>::RB * XCfg<N>::T)
k_xinv(FluidGeom g, const double2 *__restrict__ spec, double *out, int ncomp,
       const double2 *__restrict__ twN, const double2 *__restrict__ twM, long long *flag,
       const long long *dev_n, long long n) {
  constexpr int M = N / 2, RB = XCfg<N>::RB, T = XCfg<N>::T, LD = Plan<M>::LD;
  extern __shared__ double2 sm[];
  const int z = blockIdx.y, y0 = blockIdx.x * RB;
  const int t = threadIdx.x % T, pencil = threadIdx.x / T;
  const int row = pencil % RB, comp = pencil / RB;
  const double2 *in = spec + (((size_t)comp * g.N3 + z) * g.N2 + (y0 + row)) * g.P;
  const size_t V = (size_t)g.V;
  double2 *o2 = reinterpret_cast<double2 *>(out + comp * V + ((size_t)z * g.N2 + (y0 + row)) * N);
  auto ld = [&](int e) -> double2 {
    double2 Xk = in[e], Xm = in[M - e];
    if (e == 0) { Xk.y = 0.0; Xm.y = 0.0; }      // X_0, X_{N/2} are real
    const double2 A = make_double2(Xk.x + Xm.x, Xk.y - Xm.y);
    const double2 B = make_double2(Xk.x - Xm.x, Xk.y + Xm.y);
    const double2 cB = cmul(cconj(__ldg(&twN[e])), B);
    return make_double2(A.x - cB.y, A.y + cB.x);
  };
  bool bad = false;
  auto st = [&](int k, double2 v) {
    bad |= !(isfinite(v.x) && isfinite(v.y));
    o2[k] = v;
  };
  fft_io<M, +1, false, true>(sm + pencil * LD, t, twM, ld, st);
  if (flag && __syncthreads_or(bad) && threadIdx.x == 0) {
    const long long s = dev_n ? *dev_n : n;
    atomicMin(flag, s);
  }
}

template <int N>
static cudaError_t launch_xinv_n(const FluidGeom &g, const double2 *spec, double *out,
                                 int ncomp, const double2 *twN, const double2 *twM,
                                 long long *flag, const long long *dev_n, long long n,
                                 cudaStream_t s) {
  using X = XCfg<N>;
  if (g.N2 % X::RB) return cudaErrorInvalidValue;
  dim3 grid(g.N2 / X::RB, g.N3);
  const size_t smem = (size_t)ncomp * X::RB * Plan<N / 2>::LD * sizeof(double2);
  k_xinv<N><<<grid, ncomp * X::RB * X::T, smem, s>>>(g, spec, out, ncomp, twN, twM, flag,
                                                     dev_n, n);
  return cudaGetLastError();
}

// rows per x-pass tile (XCfg<N1>::RB): ib_create3 requires N2 to be a multiple of it
int xfwd_rows(int N1) {
  switch (N1) {
    case 8: return XCfg<8>::RB;      case 16: return XCfg<16>::RB;    case 32: return XCfg<32>::RB;
    case 64: return XCfg<64>::RB;    case 128: return XCfg<128>::RB;  case 256: return XCfg<256>::RB;
    case 512: return XCfg<512>::RB;  default: return 0;
  }
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
                        unsigned *rowflag, const double *in, double *r_out, double2 *spec,
                        const double2 *twN, const double2 *twM, const XMapsU *um,
                        cudaStream_t s) {
#define CALL(n) launch_xfwd_n<n>(g, mode, u, F, rowflag, in, r_out, spec, twN, twM, um, s)
  IBK_DISPATCH_N(g.N1, CALL)
#undef CALL
}

cudaError_t launch_ypass(const FluidGeom &g, int sign, const double2 *in, int in_layout,
                         double2 *out, int out_layout, int ncomp, const double2 *twN,
                         cudaStream_t s) {
#define CALL(n) launch_ypass_n<n>(g, sign, in, in_layout, out, out_layout, ncomp, twN, s)
  IBK_DISPATCH_N(g.N2, CALL)
#undef CALL
}

cudaError_t launch_zpass(const FluidGeom &g, int mode, double2 *spec, double2 *pspec,
                         const double2 *twN, const Sym &sym, cudaStream_t s) {
#define CALL(n) launch_zpass_n<n>(g, mode, spec, pspec, twN, sym, s)
  IBK_DISPATCH_N(g.N3, CALL)
#undef CALL
}

cudaError_t launch_xinv(const FluidGeom &g, const double2 *spec, double *out, int ncomp,
                        const double2 *twN, const double2 *twM, long long *flag,
                        const long long *dev_n, long long n, cudaStream_t s) {
#define CALL(n_) launch_xinv_n<n_>(g, spec, out, ncomp, twN, twM, flag, dev_n, n, s)
  IBK_DISPATCH_N(g.N1, CALL)
#undef CALL
}

// TMA descriptors of a u-shaped array [3][N3][N2][N1]: RB-row and 1-row boxes of x rows.
bool xfwd_encode_u(const FluidGeom &g, const double *u, XMapsU *m) {
  m->ok = false;
  const int N = g.N1;
  if (N > 512 || N < 16) return false;     // rows >= 128 B (smem alignment)
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                       &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return false;
  auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  int rb = 0;
  switch (N) {
    case 8: rb = XCfg<8>::RB; break;      case 16: rb = XCfg<16>::RB; break;
    case 32: rb = XCfg<32>::RB; break;    case 64: rb = XCfg<64>::RB; break;
    case 128: rb = XCfg<128>::RB; break;  case 256: rb = XCfg<256>::RB; break;
    case 512: rb = XCfg<512>::RB; break;
    default: return false;
  }
  void *base = const_cast<double *>(u);
#ifndef IBK_X512TMA
#define IBK_X512TMA 1
#endif
  if (N > 256) {          // a TMA box row is at most 256 elements: (256, 2 halves, row) view
    if (!IBK_X512TMA) return false;
    cuuint64_t d3[3] = {256, 2, (cuuint64_t)3 * g.N2 * g.uN3};
    cuuint64_t s3[2] = {256 * 8, (cuuint64_t)N * 8};
    cuuint32_t b3[3] = {256, 2, (cuuint32_t)rb}, b31[3] = {256, 2, 1}, e3[3] = {1, 1, 1};
    if (fn(&m->rows, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, d3, s3, b3, e3,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
    if (fn(&m->row1, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, d3, s3, b31, e3,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
    m->ok = true;
    return true;
  }
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)3 * g.N2 * g.uN3}, strides[1] = {(cuuint64_t)N * 8};
  cuuint32_t box[2] = {(cuuint32_t)N, (cuuint32_t)rb}, box1[2] = {(cuuint32_t)N, 1u}, es[2] = {1, 1};
  if (fn(&m->rows, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (fn(&m->row1, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box1, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  m->ok = true;
  return true;
}

template <int N>
static cudaError_t set_attrs_n() {
  const int big = 200 * 1024;
  cudaError_t e = cudaSuccess;
#define SETA(K) if (e == cudaSuccess) e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, big)
  SETA((k_xfwd<N, 0>)); SETA((k_xfwd<N, 1>)); SETA((k_xfwd<N, 2>));
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
