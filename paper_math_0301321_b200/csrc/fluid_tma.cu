// fluid_tma.cu — the strided FFT passes of step 3 (PAPER.md 692-695) as TMA-fed column-tile
// kernels for N in [64, 512]:
//
//   MODE_Z    : S2 -> S2   forward z FFT, per-mode implicit-viscosity + projection solve
//               (eq:discreteNS1-2; DESIGN.md §2 S3c, readings Z6/Z22), inverse z FFT
//   MODE_YFWD : S1 -> S2   forward y FFT (transposing [comp][z][y][kx] -> [comp][ky][z][kx])
//   MODE_YINV : S2 -> S1   inverse y FFT (the transpose back)
//   MODE_ZFWD : S2 -> S2   forward z FFT only (ib_debug_fft)
//   MODE_ZINV : S2 -> S2   inverse z FFT only (the pressure spectrum written by MODE_Z)
//
// A tile is 8 consecutive kx columns (128 bytes per row) x N rows x 3 components.  One
// producer warp streams tiles HBM -> smem with cp.async.bulk.tensor (SWIZZLE_128B: element
// (row e, column c) sits at chunk c ^ (e & 7) of its 128-byte row) into a ring of STAGES
// buffers and drains finished tiles smem -> HBM with bulk tensor stores; 3*8*T consumer
// threads (column fastest, so the 8 lanes of every quarter-warp touch 8 distinct 16-byte
// bank groups in every access) transform the tile IN PLACE with the Stockham passes of
// fft.cuh (register DFT-16, barrier, store).  Loads, compute and stores of consecutive
// tiles overlap; nothing is staged in registers across tiles.
#include <cstdio>

#include "fft.cuh"
#include "ib_internal.cuh"
#include "tma.cuh"

namespace ibk {

enum { MODE_Z = 0, MODE_YFWD = 1, MODE_YINV = 2, MODE_ZFWD = 3, MODE_ZINV = 4 };
#ifndef IBK_YG256
#define IBK_YG256 1
#endif
#ifndef IBK_ZG128
#define IBK_ZG128 4
#endif

// Column tile geometry: C columns (C = 8 -> 128-byte rows, SWIZZLE_128B; C = 4 -> 64-byte
// rows, SWIZZLE_64B), N rows, NC components (3 when the tile is solved, 1 for the y passes),
// S ring stages; G consumer groups work on consecutive tiles independently (own named
// barrier), so one group's barrier waits overlap another group's arithmetic.
template <int N, int C_, int G_, int NC_, int S_>
struct CT {
  static constexpr int C = C_, G = G_, NC = NC_, STAGES = S_;
  static constexpr int T = Plan<N>::T;                 // threads per pencil
  static constexpr int NTG = NC * C * T;               // consumer threads per group
  static constexpr int NT = G * NTG;                   // consumer threads
  static constexpr int NTHR = NT + 32;                 // + one producer warp
  static constexpr int TILE = N * C;                   // complex per component
  static constexpr uint32_t STAGE_BYTES = (uint32_t)NC * TILE * 16u;
  static constexpr int BOXR = N < 256 ? N : 256;       // TMA box rows (<= 256)
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024;
  static_assert(NTG % 32 == 0, "named barriers need whole warps");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};
// Per pass: the y passes touch the large-pitch side of S2 (ky stride N*P*16 B), where
// 128-byte rows are needed for DRAM efficiency (tools/membench.cu), and transform each
// component independently (NC = 1, more, smaller stages); the z passes need the 3
// components of a mode together (NC = 3) and stay on the small pitch, where 64-byte rows
// stream at full rate.
template <int N, int MODE> struct ColCfg {
  static constexpr bool ZM = MODE == MODE_Z || MODE == MODE_ZFWD || MODE == MODE_ZINV;
  static constexpr int C = (ZM && N >= 128) ? 4 : 8;
#ifdef IBK_Y256_NC3   // dev experiment: y passes at N = 256 with 3-component tiles
  static constexpr int NC = (ZM || N == 256) ? 3 : 1;
  static constexpr int G = ZM ? (N == 128 || N == 256 ? 2 : 1) : (N >= 512 ? 1 : (N == 256 ? 1 : 4));
#else
  static constexpr int NC = ZM ? 3 : 1;
// z pass at N3 = 256: 2 consumer groups of 6 warps, 4 stages (218 us; 3 groups with the
// 3 stages the stage/group rule below allows: 226 us; 1 group 316 us)
#ifndef IBK_ZG256
#define IBK_ZG256 2
#endif
  static constexpr int G = ZM ? (N == 256 ? IBK_ZG256 : (N == 128 ? IBK_ZG128 : (N < 128 ? 4 : 1)))
                              : (N >= 512 ? 1 : (N == 256 ? IBK_YG256 : 4));
#endif
  static constexpr size_t SB = (size_t)NC * N * C * 16;
  static constexpr int S0 = (int)((200 * 1024) / SB);
  // Each stage must always be consumed by the same group (S a multiple of G): a group only
  // waits for round r + 1 of a stage after it consumed round r itself.  Otherwise a group
  // could test a stage's mbarrier parity while the round before it (owned by another group)
  // has not completed yet, and the parity test would pass two phases early.
  static constexpr int S1 = S0 > 2 * G + 1 ? 2 * G + 1 : S0;
  static constexpr int S = S1 >= G ? (S1 / G) * G : S1;
  static_assert(S % G == 0, "stages per consumer group");
  using K = CT<N, C, G, NC, S>;
};

// Mixed-radix walk over tiles t = (c * W + w) * NB + x (x fastest) advancing by a fixed
// stride: one division at the start, carries afterwards (NB, W are runtime values).
struct Walk {
  int x, w, c, dx, dw, dc, NB, W;
  __device__ Walk(int tile, int stride, int NB_, int W_) : NB(NB_), W(W_) {
    x = tile % NB; w = (tile / NB) % W; c = tile / (NB * W);
    dx = stride % NB; dw = (stride / NB) % W; dc = stride / (NB * W);
  }
  __device__ __forceinline__ void next() {
    x += dx;
    int cy = 0;
    if (x >= NB) { x -= NB; cy = 1; }
    w += dw + cy;
    cy = 0;
    if (w >= W) { w -= W; cy = 1; }
    c += dc + cy;
  }
};

// Tile element (row e, column col) in 16-byte units under the TMA swizzle of the C-wide box.
template <int C>
__device__ __forceinline__ int swz(int e, int col) {
  if constexpr (C == 8) return e * 8 + (col ^ (e & 7));
  else return e * 4 + (col ^ ((e >> 1) & 3));
}

// Pass store with a per-thread pair flip: a thread with odd t writes its outputs (r, r+1)
// in the order (r+1, r), so for NS = 1 passes the 2 pencil jobs of a quarter-warp (4-column
// tiles) hit rows of different parity -> distinct 64-byte-swizzle bank groups.
template <int L, int PASS, class STF>
__device__ __forceinline__ void pass_st_flip(const double2 *v, int t, STF st) {
  using I = PassI<L, PASS>;
  const bool f = t & 1;
#pragma unroll
  for (int q = 0; q < I::J; ++q) {
    const int j = t + q * Plan<L>::T;
    const int base = (j / I::NS) * I::NS * I::R + (j % I::NS);
#pragma unroll
    for (int r = 0; r < I::R; r += 2) {
      const double2 a = v[q * I::R + r], b = v[q * I::R + r + 1];
      st(base + (f ? r + 1 : r) * I::NS, f ? b : a);
      st(base + (f ? r : r + 1) * I::NS, f ? a : b);
    }
  }
}

#ifndef IBK_LASTBAR
#define IBK_LASTBAR 0
#endif
// In-place length-L Stockham transform of the pencil accessed by A(e) (a double2&), by its
// T threads; every thread of the consumer group must call it (named barrier BAR, NTG).
// FUSE: at L = 512 fold the radix-2 first pass into the second pass's loads (z modes: the
// z solve 2240 -> 2080 us at 512^3; the y passes, whose 128-byte-row tiles are read by more
// threads per pencil element, lost 170-290 us with it)
template <int L, int SIGN, int C, bool POW = false, bool FUSE = false, class ACC, class TW>
__device__ __forceinline__ void fft_inplace(ACC A, int t, TW tw,
                                            int bar, int ntg) {
  double2 v[Plan<L>::RMAX];
  auto ld = [&](int e) { return A(e); };
  auto st = [&](int e, double2 x) { A(e) = x; };
#ifndef IBK_FUSE2
#define IBK_FUSE2 1
#endif
  if constexpr (FUSE && IBK_FUSE2 && Plan<L>::NPASS == 3 && PassI<L, 0>::R == 2) {
    // L = 512 (radix 2, 16, 16): the radix-2 pass is folded into the loads of the second
    // pass — its output at e is x[e/2] +- x[e/2 + L/2] (no twiddles at NS = 1) — so the
    // pencil makes one shared-memory round trip less and two barriers fewer
    auto ld2 = [&](int e) {
      const double2 a = A(e >> 1), b = A((e >> 1) + L / 2);
      return (e & 1) ? csub(a, b) : cadd(a, b);
    };
    pass_lc<L, SIGN, 1, POW>(v, t, tw, ld2);
    named_bar(bar, ntg);
    pass_st<L, 1>(v, t, st);
    named_bar(bar, ntg);
    pass_lc<L, SIGN, 2, POW>(v, t, tw, ld);
    if (IBK_LASTBAR) named_bar(bar, ntg);
    pass_st<L, 2>(v, t, st);
    named_bar(bar, ntg);
    return;
  }
  pass_lc<L, SIGN, 0>(v, t, tw, ld);
  named_bar(bar, ntg);
  if constexpr (C == 4 && PassI<L, 0>::NS == 1 && Plan<L>::NPASS > 1) pass_st_flip<L, 0>(v, t, st);
  else pass_st<L, 0>(v, t, st);
  named_bar(bar, ntg);
  // The last pass is thread-local in place (job j reads and writes j + r NS, NS = L / R), so
  // its stores need no barrier after its loads; the other passes scatter across threads.
  if constexpr (Plan<L>::NPASS > 1) {
    pass_lc<L, SIGN, 1, POW>(v, t, tw, ld);
    if (Plan<L>::NPASS > 2 || IBK_LASTBAR) named_bar(bar, ntg);
    pass_st<L, 1>(v, t, st);
    named_bar(bar, ntg);
  }
  if constexpr (Plan<L>::NPASS > 2) {
    pass_lc<L, SIGN, 2, POW>(v, t, tw, ld);
    if (IBK_LASTBAR) named_bar(bar, ntg);
    pass_st<L, 2>(v, t, st);
    named_bar(bar, ntg);
  }
}

template <int N, int MODE>
__global__ void __launch_bounds__(ColCfg<N, MODE>::K::NTHR, 1)
k_colfft(FluidGeom g, const __grid_constant__ CUtensorMap map_ld,
         const __grid_constant__ CUtensorMap map_st, double2 *pspec,
         const double2 *__restrict__ twN, Sym sym, const __grid_constant__ PeerMaps peers) {
  using K = typename ColCfg<N, MODE>::K;
  constexpr int C = K::C, G = K::G, T = K::T, NTG = K::NTG, NT = K::NT, S = K::STAGES;
  constexpr int NC = K::NC, BR = K::BOXR;
  // N = pencil length (N2 for the y modes, N3 for the z modes); W = the other lattice
  // dimension the tiles walk (z planes for y, ky for z); kx in [0, M], M = N1/2
  constexpr bool YM = MODE == MODE_YFWD || MODE == MODE_YINV;
  const int M = g.M, NB = (M + 1 + C - 1) / C, W = YM ? g.N3 : g.N2;
  extern __shared__ __align__(1024) double2 smraw[];
  __shared__ uint64_t full[S], done[S];
  // 1024-byte aligned ring (swizzle atoms); offset arithmetic on the __shared__ array
  // keeps every tile access an LDS/STS (a uintptr_t round trip would make them generic)
  double2 *stage0 = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u) / 16u;
  const int ntiles = NB * W * (NC == 1 ? 3 : 1);      // NC = 1: (kx block, w, comp) tiles
  // The forward y pass walks each component's planes top-down: the x forward pass wrote
  // them bottom-up, so the last-written planes are read while still in L2 (-1 us at 256^3;
  // walking planes outermost with the components inside was +2.4 us per y pass).
#ifndef IBK_L2ORDER
#define IBK_L2ORDER 1
#endif
  constexpr bool YREV = IBK_L2ORDER && MODE == MODE_YFWD;
  const int WW = W;
  auto tile_w = [&](const Walk &t) {
    if constexpr (YREV) return W - 1 - t.w;
    else return t.w;
  };
  auto tile_c = [&](const Walk &t) { return t.c; };
  // z symbols (sin and sin^2 terms along the pencil) staged once: the solve reads them per
  // element, an L1/L2 latency the loop would otherwise expose on every iteration
  __shared__ double symz[MODE == MODE_Z ? 2 * N : 1];
  if constexpr (MODE == MODE_Z)
    for (int k = threadIdx.x; k < N; k += blockDim.x) { symz[k] = sym.sz[k]; symz[N + k] = sym.lz[k]; }
  // z modes: twiddles staged likewise (one copy per persistent CTA; 2511 -> 2316 us at
  // 512^3, neutral at 256^3).  The y modes keep the read-only global path: their shared
  // memory is busier and staged twiddles slowed them (139 -> 174 us at 256^3).
  constexpr bool ZM = ColCfg<N, MODE>::ZM;
  __shared__ double2 tws[ZM ? N : 1];
  if constexpr (ZM)
    for (int k = threadIdx.x; k < N; k += blockDim.x) tws[k] = twN[k];
  // y modes with a 2-pass plan: the pass-1 job of a consumer thread is its own t (J = 1), so
  // its 15 twiddles are read once into registers (their per-tile table reads were the
  // largest stall of these passes); z modes read a shared-memory copy with power products
#ifndef IBK_YREGTW
#define IBK_YREGTW 1
#endif
  constexpr bool YREG = IBK_YREGTW && !ZM && Plan<N>::NPASS == 2 && PassI<N, 1>::J == 1 &&
                        PassI<N, 1>::R == 16;
  const int t_cons = (threadIdx.x % K::NTG) / C % K::T;
  const auto tw = [&]() {
    if constexpr (ZM) return SmemTw{tws};
    else if constexpr (YREG)
      return make_regtw16<(MODE == MODE_YINV) ? +1 : -1>(
          twN, (t_cons % PassI<N, 1>::NS) * (N / (PassI<N, 1>::NS * 16)));
    else return twN;
  }();
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&done[s], 1); }
    fence_mbar_init();
  }
  __syncthreads();

  // 2-D maps address rows (comp*N + w)*N + r; 3-D maps (x, w, comp*N + r) — see encode()
  constexpr bool LD3 = MODE == MODE_YINV, ST3 = MODE == MODE_YFWD;
  constexpr bool SLABZ = MODE == MODE_Z;                 // slab z pass: 5-D maps
  if (threadIdx.x >= NT) {                               // ---------------- producer warp
    if (threadIdx.x == NT) {
      prefetch_tmap(&map_ld);
      prefetch_tmap(&map_st);
      // tile -> (x offset in doubles, w = ky or z, first component); boxes of BR rows
      auto load = [&](const Walk &t, int s) {
        const int x = 2 * C * t.x, w = tile_w(t), c0 = NC == 1 ? tile_c(t) : 0;
        double2 *b = stage0 + (size_t)s * NC * K::TILE;
        mbar_expect_tx(&full[s], K::STAGE_BYTES);
        for (int c = 0; c < NC; ++c)
          for (int r0 = 0; r0 < N; r0 += BR) {
            double2 *d = b + c * K::TILE + r0 * C;
            if (LD3) tma_load_3d(d, &map_ld, x, w, (c0 + c) * N + r0, &full[s]);
            else if (SLABZ && g.slab)   // received slab blocks [comp][src][ky][z_src][kx]
              tma_load_5d(d, &map_ld, x, 0, w, r0 / g.L, c0 + c, &full[s]);
            else     tma_load_2d(d, &map_ld, x, ((c0 + c) * W + w) * N + r0, &full[s]);
          }
      };
      auto store = [&](const Walk &t, int s) {
        const int x = 2 * C * t.x, w = tile_w(t), c0 = NC == 1 ? tile_c(t) : 0;
        const double2 *b = stage0 + (size_t)s * NC * K::TILE;
        if ((MODE == MODE_YFWD || MODE == MODE_Z) && peers.P) {   // fused slab transposes
          const int R = peers.rows;
          for (int c = 0; c < NC; ++c)
            for (int d = 0; d < peers.P; ++d) {
              if (MODE == MODE_YFWD)   // ky rows [d Ky, (d+1) Ky) -> rank d's Z [c0][r][.][w]
                tma_store_4d(&peers.m[d], x, w, 0, c0, b + (c * N + d * R) * C);
              else                     // kz rows [d L, (d+1) L) -> rank d's S2 [c][r][w][.]
                tma_store_4d(&peers.m[d], x, 0, w, c, b + c * K::TILE + d * R * C);
            }
          bulk_commit();
          return;
        }
        for (int c = 0; c < NC; ++c)
          for (int r0 = 0; r0 < N; r0 += BR) {
            const double2 *d = b + c * K::TILE + r0 * C;
            if (ST3) tma_store_3d(&map_st, x, w, (c0 + c) * N + r0, d);
            else if (SLABZ && g.slab) tma_store_5d(&map_st, x, 0, w, r0 / g.L, c0 + c, d);
            else     tma_store_2d(&map_st, x, ((c0 + c) * W + w) * N + r0, d);
          }
        bulk_commit();
      };
      Walk lw(blockIdx.x, gridDim.x, NB, WW), sw(blockIdx.x, gridDim.x, NB, WW);
      int i = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
        const int s = i % S;
        if (i >= S) {                                    // slot s held tile i - S
          mbar_wait(&done[s], ((i / S) - 1) & 1);
          store(sw, s);
          sw.next();
          bulk_wait_read0();                             // smem of slot s read out
        }
        load(lw, s);
        lw.next();
      }
      for (int k = i - S < 0 ? 0 : i - S; k < i; ++k) {  // drain the last tiles
        const int s = k % S;
        mbar_wait(&done[s], (k / S) & 1);
        store(sw, s);
        sw.next();
      }
      bulk_wait0();
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  const int grp = threadIdx.x / NTG, gtid = threadIdx.x % NTG, bar = 1 + grp;
  const int col = gtid % C, t = (gtid / C) % T, comp = gtid / (C * T);
  int i = grp;
  Walk cw(blockIdx.x + grp * gridDim.x, G * gridDim.x, NB, WW);
  const double cdt = g.rho / g.dt, invV = 1.0 / (double)g.Vg;  // solve constants (MODE_Z)
  for (int tile = blockIdx.x + grp * gridDim.x; tile < ntiles; tile += G * gridDim.x, i += G, cw.next()) {
    const int s = i % S;
    if (s % G != grp) __trap();                          // ring-ownership rule (ColCfg)
    // MODE_Z: the tile's x / y symbols are read before the stage wait and the forward FFT,
    // so their L1/L2 latency overlaps them instead of stalling the solve
    const int kx0 = C * cw.x, ky = cw.w;
    const int kyg = g.ky0 + ky;                          // global ky (slab z pass: offset)
    static_assert(NTG % C == 0, "solve mapping");
    const int c = gtid % C, kx = kx0 + c;                // column c = gtid % C per thread
    const bool live = kx <= M;
    double sy = 0.0, ly = 0.0, sx = 0.0, lx = 0.0;
    auto load_sym = [&]() {
      sy = sym.sy[kyg]; ly = sym.ly[kyg];
      if (live) { sx = sym.sx[kx]; lx = sym.lx[kx]; }
    };
#ifndef IBK_ZHOIST
#define IBK_ZHOIST 1
#endif
    if (MODE == MODE_Z && IBK_ZHOIST) load_sym();
    mbar_wait(&full[s], (i / S) & 1);
    double2 *buf = stage0 + (size_t)s * NC * K::TILE;
    double2 *pc = buf + comp * K::TILE;
    auto A = [pc, col](int e) -> double2 & { return pc[swz<C>(e, col)]; };
    if (MODE == MODE_Z) {
      fft_inplace<N, -1, C, true, true>(A, t, tw, bar, NTG);  // z: power twiddles
      if (!IBK_ZHOIST) load_sym();
      const bool ny = (kyg == 0) || (2 * kyg == g.N2g);
      const double lxy = lx + ly;
      const bool nxy = ny && (kx == 0 || kx == M);
      // û = (r̂ - s (s.r̂)/|s|^2)/d, p̂ = -i (s.r̂)/|s|^2; null modes (Z6): û = r̂/d
      auto solve = [&](int kz, double2 *q0, double2 r0, double2 r1, double2 r2) {
        double2 *q1 = q0 + K::TILE, *q2 = q1 + K::TILE;
        const double sz = symz[kz];
        const double d = cdt + g.mu * (lxy + symz[N + kz]);
        const bool nul = nxy && (kz == 0 || 2 * kz == N);
        if (nul) {                                       // reading Z6
          const double inv = invV / d;
          *q0 = cscale(r0, inv); *q1 = cscale(r1, inv); *q2 = cscale(r2, inv);
          if (pspec) pspec[((size_t)ky * N + kz) * g.P + kx] = make_double2(0.0, 0.0);
        } else {
          // one division: w = 1/(d |s|^2) gives 1/d = w |s|^2 and 1/|s|^2 = w d
          const double s2 = sx * sx + sy * sy + sz * sz;
          const double w = rcp_pos(d * s2);
          const double is2 = w * d, inv = invV * (w * s2);
          const double2 q = make_double2((sx * r0.x + sy * r1.x + sz * r2.x) * is2,
                                         (sx * r0.y + sy * r1.y + sz * r2.y) * is2);
          *q0 = make_double2((r0.x - sx * q.x) * inv, (r0.y - sx * q.y) * inv);
          *q1 = make_double2((r1.x - sy * q.x) * inv, (r1.y - sy * q.y) * inv);
          *q2 = make_double2((r2.x - sz * q.x) * inv, (r2.y - sz * q.y) * inv);
          if (pspec) pspec[((size_t)ky * N + kz) * g.P + kx] = make_double2(q.y * invV, -q.x * invV);
        }
      };
      for (int kz = gtid / C; live && kz < N; kz += NTG / C) {
        double2 *q0 = buf + swz<C>(kz, c);
        solve(kz, q0, q0[0], q0[K::TILE], q0[2 * K::TILE]);
      }
      named_bar(bar, NTG);
      fft_inplace<N, +1, C, true, true>(A, t, tw, bar, NTG);
    } else {
      fft_inplace<N, (MODE == MODE_YINV || MODE == MODE_ZINV) ? +1 : -1, C, ZM, ZM>(A, t, tw, bar, NTG);
    }
    fence_proxy_async();                                 // generic writes -> TMA store
    named_bar(bar, NTG);
    if (gtid == 0) mbar_arrive(&done[s]);
  }
}

// ------------------------------------------------------------------ tensor maps
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// 2-D view: rows of one spectrum array, row r = (comp*N + w)*N + e; 3-D view of S2:
// (x, z, comp*N + ky).  Inner dimension in doubles (2 per complex, N/2+1 complex valid,
// row pitch P complex); boxes are 2C doubles (C*16 bytes) x N rows with the matching
// swizzle (C = 8: 128 B, C = 4: 64 B).  Columns past N/2 are zero-filled on load and
// clipped on store.
// rank 2: rows of one spectrum array viewed as [3 * N_outer * L][row], row index
//         (comp*W + w)*L + e (S1: W = N3, L = N2; S2: W = N2, L = N3 — same row count);
// rank 3: S2 as (x, z, comp*N2 + ky).  Boxes: 2C doubles x min(L, 256) rows.
static bool encode(CUtensorMap *m, void *base, int rank, const FluidGeom &g, int C, int L) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3], strides[2];
  cuuint32_t box[3], es[3] = {1, 1, 1};
  dims[0] = (cuuint64_t)2 * (g.M + 1);
  strides[0] = (cuuint64_t)g.P * 16;
  box[0] = (cuuint32_t)(2 * C);
  const cuuint32_t br = (cuuint32_t)(L < 256 ? L : 256);
  if (rank == 2) {
    dims[1] = (cuuint64_t)3 * g.N2 * g.N3;
    box[1] = br;
  } else {
    dims[1] = (cuuint64_t)g.N3;              // z
    dims[2] = (cuuint64_t)3 * g.N2;          // comp*N2 + ky
    strides[1] = (cuuint64_t)g.N3 * g.P * 16;
    box[1] = 1;
    box[2] = br;
  }
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  C == 8 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int zcols(int N3) { return N3 >= 128 ? 4 : 8; }   // = ColCfg<N3, MODE_Z>::C

// Slab z pass: the received transpose blocks Z [comp][src][ky][z_src][kx]
// (P source ranks of L planes each, Ky local ky rows, pitch gz.P complex) as a 5-D map
// (x, z_src, ky, src, comp); a box {2C, L, 1, BR/L, 1} is BR consecutive rows kz = src L + z.
bool colfft_encode_slabz(const FluidGeom &gz, double2 *Z, int P, CUtensorMap *m) {
  auto fn = encode_fn();
  const int N = gz.N3, L = gz.L, C = zcols(N);
  const int br = N < 256 ? N : 256;
  if (!fn || !colfft_supported(N) || L * P != N || br % L) return false;
  const cuuint64_t row = (cuuint64_t)gz.P * 16;
  cuuint64_t dims[5] = {(cuuint64_t)2 * (gz.M + 1), (cuuint64_t)L, (cuuint64_t)gz.N2,
                        (cuuint64_t)P, 3};
  cuuint64_t strides[4] = {row, row * L, row * L * gz.N2, row * L * gz.N2 * P};
  cuuint32_t box[5] = {(cuuint32_t)(2 * C), (cuuint32_t)L, 1, (cuuint32_t)(br / L), 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, Z, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE,
            C == 8 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Peer block view: buffer [comp][P][Ky][L][kx] (pitch gz.P complex), block `blk` of the P
// axis, as (x, z_l, ky_l, comp) with the P axis folded into the comp stride.
bool colfft_encode_peer(const FluidGeom &gz, double2 *buf, int P, int blk, int C, int zbox,
                        int kybox, CUtensorMap *m) {
  auto fn = encode_fn();
  const int L = gz.L, Ky = gz.N2;
  if (!fn || P < 1 || P > MAX_PEERS || blk < 0 || blk >= P) return false;
  const cuuint64_t row = (cuuint64_t)gz.P * 16;
  cuuint64_t dims[4] = {(cuuint64_t)2 * (gz.M + 1), (cuuint64_t)L, (cuuint64_t)Ky, 3};
  cuuint64_t strides[3] = {row, row * L, row * L * Ky * P};
  cuuint32_t box[4] = {(cuuint32_t)(2 * C), (cuuint32_t)zbox, (cuuint32_t)kybox, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  double2 *base = buf + (size_t)blk * Ky * L * gz.P;
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE,
            C == 8 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool colfft_supported(int N) { return N >= 64 && N <= 512; }

bool colfft_encode_s2(const FluidGeom &g, double2 *base, CUtensorMap *m) {
  return colfft_supported(g.N3) && encode(m, base, 2, g, zcols(g.N3), g.N3);
}

// y passes need N2 in [64, 512] (maps.y_ok), z passes N3 in [64, 512] (maps.z_ok)
cudaError_t colfft_make_maps(const FluidGeom &g, double2 *spec, double2 *spec2, TmaMaps *m) {
  m->y_ok = m->z_ok = false;
  if (colfft_supported(g.N2)) {
    if (!encode(&m->s1_2d, spec, 2, g, 8, g.N2) || !encode(&m->s2_3d, spec2, 3, g, 8, g.N2))
      return cudaErrorInvalidValue;
    m->y_ok = true;
  }
  if (colfft_supported(g.N3)) {
    if (!encode(&m->s2_2d, spec2, 2, g, zcols(g.N3), g.N3)) return cudaErrorInvalidValue;
    m->z_ok = true;
  }
  return cudaSuccess;
}

template <class Kern>
static int one_per_sm_grid(Kern k, int threads, size_t smem, int ntiles) {
  int per = 0;
  const int nsm = sm_count();
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, threads, smem);
  if (per < 1) per = 1;
  return ntiles < per * nsm ? ntiles : per * nsm;
}

template <int N, int MODE>
static cudaError_t launch_colfft_n(const FluidGeom &g, const CUtensorMap &ld,
                                   const CUtensorMap &st, double2 *pspec, const double2 *twN,
                                   const Sym &sym, cudaStream_t s, const PeerMaps &peers) {
  using K = typename ColCfg<N, MODE>::K;
  static PerDeviceOnce attr;
  const int dev = current_device();
  if (!attr.done(dev)) {
    cudaError_t e = cudaFuncSetAttribute(k_colfft<N, MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM);
    if (e != cudaSuccess) return e;
    attr.mark(dev);
  }
  constexpr bool YM = MODE == MODE_YFWD || MODE == MODE_YINV;
  const int NB = (g.M + 1 + K::C - 1) / K::C, W = YM ? g.N3 : g.N2;   // tiles per w, w range
  const int grid = one_per_sm_grid(k_colfft<N, MODE>, K::NTHR, K::SMEM, NB * W * (K::NC == 1 ? 3 : 1));
  k_colfft<N, MODE><<<grid, K::NTHR, K::SMEM, s>>>(g, ld, st, pspec, twN, sym, peers);
  return cudaGetLastError();
}

template <int N>
static cudaError_t colfft_n(const FluidGeom &g, int mode, const TmaMaps &m, double2 *pspec,
                            const double2 *twN, const Sym &sym, cudaStream_t s) {
  if constexpr (N >= 64 && N <= 512) {
    const PeerMaps none{};
    if (mode == MODE_ZINV) return launch_colfft_n<N, MODE_ZINV>(g, m.s2_2d, m.s2_2d, nullptr, twN, sym, s, none);
    if (mode == MODE_ZFWD) return launch_colfft_n<N, MODE_ZFWD>(g, m.s2_2d, m.s2_2d, nullptr, twN, sym, s, none);
    if (mode == MODE_Z) return launch_colfft_n<N, MODE_Z>(g, m.s2_2d, m.s2_2d, pspec, twN, sym, s, m.peers);
    if (mode == MODE_YFWD) return launch_colfft_n<N, MODE_YFWD>(g, m.s1_2d, m.s2_3d, nullptr, twN, sym, s, m.peers);
    return launch_colfft_n<N, MODE_YINV>(g, m.s2_3d, m.s1_2d, nullptr, twN, sym, s, none);
  }
  return cudaErrorInvalidValue;
}

// y modes (1, 2) transform along y (length N2), the z modes (0, 3, 4) along z (N3)
cudaError_t launch_colfft(const FluidGeom &g, int mode, const TmaMaps &m, double2 *pspec,
                          const double2 *twN, const Sym &sym, cudaStream_t s) {
  const bool ym = mode == MODE_YFWD || mode == MODE_YINV;
  if (ym ? !m.y_ok : !m.z_ok) return cudaErrorInvalidValue;
  switch (ym ? g.N2 : g.N3) {
    case 64: return colfft_n<64>(g, mode, m, pspec, twN, sym, s);
    case 128: return colfft_n<128>(g, mode, m, pspec, twN, sym, s);
    case 256: return colfft_n<256>(g, mode, m, pspec, twN, sym, s);
    case 512: return colfft_n<512>(g, mode, m, pspec, twN, sym, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ibk
