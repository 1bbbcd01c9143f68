// ib_internal.cuh — context layout and kernel launchers of the B200 IB step.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include "../../include/ib.h"

namespace ibk {

// 1/a for a positive normal a: the hardware's 20-bit estimate and two Newton steps (error
// 2^-20 -> 2^-40 -> 2^-80, i.e. the last rounding only).  The compiler's fp64 division adds
// a range check and a slow-path call; the quotients formed with this differ from IEEE
// division by at most ~2 ulp, far inside the parity tolerances.  Used by the
// z solve (one reciprocal per mode: z solve 2155 -> 2126 us at 512^3, 96.3 -> 95.3 us on the
// half-cube, unchanged at 256^3); the spring force keeps the IEEE division (no gain there).
#ifndef IBK_FASTRCP
#define IBK_FASTRCP 1
#endif
__device__ __forceinline__ double rcp_pos(double a) {
#if IBK_FASTRCP
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  double e = fma(-a, y, 1.0);
  y = fma(y, e, y);
  e = fma(-a, y, 1.0);
  return fma(y, e, y);
#else
  return 1.0 / a;
#endif
}


// Device view of the Lagrangian structure (all pointers device memory).
struct StructDev {
  const double *X;            // [np][3]
  int64_t np;
  const int *perm;            // cell-binned visiting order of the points (or null)
  const double *Xs;           // [3][np] positions in that order (SoA; with perm, else null)
  const ib_patch *patches;    // [npatch]
  int32_t npatch;
  const double *stiff;
  int64_t nd;                 // drive
  const int64_t *drive_idx;
  const double *drive_dir;    // [nd][3], or null: surface-normal drive (normal of the patch)
  double drive_amp;
  int32_t drive_period;
};

// Lattice of the fluid passes: N1 x N2 x N3 points along x, y, z (powers of two), mesh width
// h in every direction (the paper's lattice of width h, PAPER.md 632-633; anisotropic boxes
// such as its 256 x 256 x 128 half-cube, 1003-1007).
struct FluidGeom {
  int N1, N2, N3;
  int M, P;                   // M = N1/2; P = spectrum row pitch in complex (>= M+1)
  int64_t V;                  // N1 N2 N3
  double h, invh, rho, mu, dt;
  // Slab decomposition along z.  Unless slab != 0 these are
  // the identity: N2g = N2, N3g = N3, Vg = V, z0 = ky0 = uz0 = 0, uN3 = N3.  In a slab the
  // arrays above are LOCAL: N3 = L planes (x and y passes) or N2 = Ky rows (z pass).
  int N2g, N3g;               // global lattice extents along y and z
  int64_t Vg;                 // global cell count (the 1/V of the unnormalised inverse FFT)
  int z0;                     // global plane of local plane 0
  int ky0;                    // z pass: global ky of local row 0
  int uz0, uN3;               // velocity array: plane index of local plane 0; planes held
  int L;                      // planes per slab (z pass: the source-rank blocks of a pencil)
  int slab;                   // 1: no periodic wrap along z inside the local arrays
};
// Identity slab fields of a whole-lattice geometry.
inline void geom_whole(FluidGeom &g) {
  g.N2g = g.N2; g.N3g = g.N3; g.Vg = g.V;
  g.z0 = 0; g.ky0 = 0; g.uz0 = 0; g.uN3 = g.N3; g.L = g.N3; g.slab = 0;
}

// Per-axis symbols (D0 symbol s, -symbol of D+D- l) of the three lattice axes.
struct Sym {
  const double *sx, *lx, *sy, *ly, *sz, *lz;
};

// TMA descriptors of the two spectrum arrays (fluid_tma.cu), valid when ok.
// Slab decomposition with fused transposes: the y forward pass stores the Ky
// rows of its tiles bound for rank d straight into rank d's receive buffer Z (map m[d]), the
// z pass the L rows of each source rank straight back into that rank's S2 — peer stores in
// place of the two all-to-alls.  P = 0: exchange mode (local stores, caller's collectives).
constexpr int MAX_PEERS = 8;
struct PeerMaps {
  CUtensorMap m[MAX_PEERS];
  int P = 0;
  int rows = 0;          // rows of one destination block in the tile (y: Ky, z: L)
};

struct TmaMaps {
  CUtensorMap s1_2d, s2_2d, s2_3d;
  bool y_ok = false, z_ok = false;   // y passes (s1_2d, s2_3d) / z passes (s2_2d) available
  PeerMaps peers;                    // fused slab transposes (y forward / z solve), or P = 0
};

// TMA descriptors of the forward x pass (fluid.cu): u rows, RB-row and 1-row boxes.
struct XMapsU {
  CUtensorMap rows, row1;
  bool ok = false;
};
// TMA descriptors of the inverse x pass (xpass_tma.cu): S1 spectrum rows (kx < N/2 box and
// the Nyquist column).
struct XMapsS {
  CUtensorMap main, nyq;
};

enum { STAGE_FORCE_SPREAD = 0, STAGE_XFWD, STAGE_YFWD, STAGE_ZPROJ, STAGE_YINV, STAGE_XINV,
       STAGE_INTERP, STAGE_COUNT };

}  // namespace ibk

struct ib_ctx {
  ibk::FluidGeom g;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  // Eulerian state and work arrays
  double *u = nullptr;          // [3][V]
  double *F = nullptr;          // [3][V]  (kept zero between steps)
  unsigned *rowflag = nullptr;  // [N*N]: row (z,y) of F touched by the spread
  double2 *spec = nullptr;      // S1 [3][z][y][P]  (x passes)
  double2 *spec2 = nullptr;     // S2 [3][ky][z][P] (z pass)
  double2 *pspec = nullptr;     // pressure, S2 layout (lazily)
  double2 *pspec1 = nullptr;    // pressure, S1 layout (lazily)
  double *p = nullptr;          // [V] pressure output cache (lazily)
  double2 *tw[3] = {};                       // exp(-2 pi i t/N_a), per axis a = x, y, z
  double2 *twM = nullptr;                    // exp(-2 pi i t/(N1/2))
  double *sym_s[3] = {}, *sym_l[3] = {};     // per-axis symbols
  ibk::TmaMaps maps;                         // TMA column-pass descriptors (N in [64, 256])
  ibk::XMapsS smaps;                         // TMA x-inverse descriptors of spec
  ibk::XMapsU umaps;                         // TMA x-forward descriptors of u (N <= 256)
  bool xok = false;
  // Lagrangian state
  int64_t np = 0;
  double *X = nullptr;
  int *perm = nullptr;          // [np] cell-binned order (binning scratch: bincnt [V], binsum)
  double *Xs = nullptr;         // [3][np] X in perm order (coalesced reads in spread / interp)
  unsigned *bincnt = nullptr, *binsum = nullptr;
  int64_t since_bin = -1;       // steps since the last binning (-1: perm invalid)
  ib_patch *patches = nullptr;
  int32_t npatch = 0;
  double *stiff = nullptr;
  int64_t nstiff = 0;
  std::vector<ib_patch> patches_h;
  int64_t nd = 0;
  int64_t *drive_idx = nullptr;
  double *drive_dir = nullptr;  // null with nd > 0: surface-normal drive
  uint8_t *fixed = nullptr;     // [np] 1 = point never moves (window plates), or null
  double drive_amp = 0.0;
  int32_t drive_period = 1;
  // control
  int64_t n = 0;
  long long *flag = nullptr;    // device: first non-finite step (LLONG_MAX = none)
  long long *flag_h = nullptr;  // pinned
  bool want_p = false, have_p = false, timing = false, use_graph = true;
  cudaEvent_t ev[ibk::STAGE_COUNT + 1] = {};
  double stage_ms[ibk::STAGE_COUNT] = {};
  std::vector<cudaEvent_t> ev_pool;   // per-step stage events (IB_OPT_STAGE_TIMING)
  int64_t launches = 0;
  // CUDA graph of one step (rebuilt after any change of structure, drive, stream, options)
  cudaGraphExec_t graph = nullptr;        // one step
  cudaGraphExec_t graph_chunk = nullptr;  // GRAPH_CHUNK steps
  long long graph_key = -1;
  long long *dev_n = nullptr;   // device step counter (drive phase, non-finite flag)
  // slab decomposition along z (ib_slab_create): rank slab_rank of slab_P.
  // g then describes the local planes (x and y passes, spread, interp), gz the z pass over
  // the received transpose blocks; the exchange buffers belong to the caller.
  int slab_P = 0, slab_rank = 0;
  int slab_next = 0;            // next ib_slab_phase expected (0..4, cyclic)
  ibk::FluidGeom gz{};
  ibk::TmaMaps zmaps;
  double2 *s2_ext = nullptr, *z_ext = nullptr;   // [3][N2][L][P] / [3][P][Ky][L][P] complex
  double *edge_send = nullptr, *edge_recv = nullptr;
  double4 *pack_send = nullptr, *pack_recv = nullptr;
  unsigned long long *count_send = nullptr, *count_recv = nullptr;
  int64_t pack_cap = 0;
};

namespace ibk {
// Once-per-device host state (function attributes apply to the current device only; a
// second context on another GPU of the same process must set them again).
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
struct PerDeviceOnce {
  std::atomic<unsigned long long> bits{0};
  bool done(int dev) const { return dev < 64 && ((bits.load() >> dev) & 1ull); }
  void mark(int dev) { if (dev < 64) bits.fetch_or(1ull << dev); }
};
// SM count of the current device (cached per device)
inline int sm_count() {
  static std::atomic<int> cache[64];
  const int d = current_device();
  int v = d < 64 ? cache[d].load() : 0;
  if (!v) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    if (d < 64) cache[d].store(v);
  }
  return v;
}
// kernels/launchers (fluid.cu)
cudaError_t init_tables(ib_ctx *c);
int xfwd_rows(int N1);   // rows per x-pass tile: N2 must be a multiple
// twiddles and symbols of one lattice axis of length N (slab contexts: the whole z axis)
cudaError_t init_axis_table(double2 *twN, int N, double *s, double *l, double h, cudaStream_t st);
cudaError_t fluid_setup_attributes(int N);
// x pass: mode 0 = step (r from u,F; zero F), 1 = r only (write r_out), 2 = FFT of in (1 comp)
// rowflag (may be null = read all of F): per (z,y) row, set by the spread where F != 0
// um: TMA maps of `u` (tile rows streamed by TMA) or null / !ok (cp.async tile copy)
cudaError_t launch_xfwd(const FluidGeom &g, int mode, const double *u, double *F,
                        unsigned *rowflag, const double *in, double *r_out, double2 *spec,
                        const double2 *twN, const double2 *twM, const XMapsU *um,
                        cudaStream_t s);
bool xfwd_encode_u(const FluidGeom &g, const double *u, XMapsU *m);
// y pass between spectrum layouts (1 = S1 [comp][z][y][kx], 2 = S2 [comp][ky][z][kx])
cudaError_t launch_ypass(const FluidGeom &g, int sign, const double2 *in, int in_layout,
                         double2 *out, int out_layout, int ncomp, const double2 *twN,
                         cudaStream_t s);
// z pass on an S2 spectrum: mode 0 = fwd+project+inv (pressure if pspec != null, S2),
// 1 = forward only
cudaError_t launch_zpass(const FluidGeom &g, int mode, double2 *spec, double2 *pspec,
                         const double2 *twN, const Sym &sym, cudaStream_t s);
cudaError_t launch_xinv(const FluidGeom &g, const double2 *spec, double *out, int ncomp,
                        const double2 *twN, const double2 *twM, long long *flag,
                        const long long *dev_n, long long n, cudaStream_t s);
// TMA column passes (fluid_tma.cu): mode 0 = z fwd+solve+inv on S2 (pressure to pspec if
// non-null; p^ in (ky, kz, kx) order), 1 = y fwd S1->S2, 2 = y inv S2->S1, 3 = z forward
// only on S2, 4 = z inverse only on S2 (uses maps.s2_2d)
bool colfft_supported(int N);
bool colfft_encode_s2(const FluidGeom &g, double2 *base, CUtensorMap *m);
bool colfft_encode_slabz(const FluidGeom &gz, double2 *Z, int P, CUtensorMap *m);
// 4-D view (x, z_l, ky_l, comp) of one [comp][P][Ky][L] block column of a peer's S2 or Z
// buffer starting at block `blk`; box {2C, zbox, kybox, 1}
bool colfft_encode_peer(const FluidGeom &gz, double2 *buf, int P, int blk, int C, int zbox,
                        int kybox, CUtensorMap *m);
cudaError_t colfft_make_maps(const FluidGeom &g, double2 *spec, double2 *spec2, TmaMaps *m);
// twN: twiddles of the pencil axis (y for modes 1-2, z for 0, 3, 4)
cudaError_t launch_colfft(const FluidGeom &g, int mode, const TmaMaps &m, double2 *pspec,
                          const double2 *twN, const Sym &sym, cudaStream_t s);
// TMA inverse x pass (xpass_tma.cu), N in [64, 256]: S1 -> out (3 components)
bool xpass_supported(int N);
bool xpass_encode_s1(const FluidGeom &g, const double2 *spec, XMapsS *m);
cudaError_t launch_xinv_tma(const FluidGeom &g, const XMapsS &m, double *out,
                            const double2 *twN, const double2 *twM, long long *flag,
                            const long long *dev_n, long long n, cudaStream_t s);
// Lagrangian kernels (lagrangian.cu)
cudaError_t launch_force(const StructDev &sd, const long long *dev_n, long long n,
                         double *f_out, cudaStream_t s);
cudaError_t launch_force_spread(const StructDev &sd, const FluidGeom &g,
                                const double *f_in, const long long *dev_n, long long n,
                                double *F, unsigned *rowflag, cudaStream_t s);
// fixed (may be null): points with fixed[i] != 0 are not moved
// pack (slab, may be null): the owned points' X^{n+1} as (x, y, z, index) records, counted
// in *pack_count
// Xs (may be null; needs perm): the perm-ordered SoA copy of X, read and kept in step
cudaError_t launch_interp(const FluidGeom &g, const double *u, double *X, int64_t np,
                          double *U_out, long long *flag, const long long *dev_n, long long n,
                          const int *perm, const uint8_t *fixed, cudaStream_t s,
                          double4 *pack = nullptr, unsigned long long *pack_count = nullptr,
                          double *Xs = nullptr);
// cell binning: perm = point indices grouped by base cell, Xs = X in that order as SoA
// (6 launches + 1 memset)
cudaError_t launch_bin(const FluidGeom &g, const double *X, int64_t np, unsigned *cnt,
                       unsigned *bsum, int *perm, double *Xs, cudaStream_t s);
cudaError_t launch_gather_xs(const double *X, const int *perm, int64_t np, double *Xs,
                             cudaStream_t s);
int bin_scan_blocks(int64_t V);
cudaError_t launch_step_inc(long long *dev_n, cudaStream_t s);
// measured on one pod, ms/step with chunks of 1 / 4 / 8 / 32 steps: cfg1 0.0509 / 0.0496 /
// 0.0516 / 0.0512, cfg2 0.0623 / 0.0606 / 0.0627 / 0.0617, cfg3 0.1559 / 0.1539 / 0.1559 /
// 0.1539, cfg4 1.148 / 1.148 / 1.151 / 1.149
#ifndef IBK_GRAPH_CHUNK
#define IBK_GRAPH_CHUNK 4
#endif
constexpr int GRAPH_CHUNK = IBK_GRAPH_CHUNK;    // steps per chunk graph (divides SORT_PERIOD)
constexpr int SORT_PERIOD = 32;   // steps between re-binnings inside ib_step
}  // namespace ibk
