/* ib.h — C-ABI of the B200 (sm_100a) immersed-boundary time step.
 *
 * The operation served is the first-order IB time step of PAPER.md §3.2 (lines 592-761):
 * given (u^n, X^n) produce (u^{n+1}, X^{n+1}) by
 *   1. the nodal Lagrangian force f^n                          (PAPER.md 610-616)
 *   2. spreading F^n = sum_q f^n(q) delta_h(x - X^n(q))          (eq:discreteF, 712-723)
 *   3. the upwind / implicit-viscosity Navier-Stokes system solved by FFT
 *                                                                (eq:discreteNS1-2, 659-695)
 *   4. X^{n+1} = X^n + dt sum_x u^{n+1}(x) delta_h(x - X^n) h^3  (eq:discreteX, 725-734)
 * with Peskin's 4-point delta_h (745-759) on a periodic N1 x N2 x N3 lattice x = h(i,j,k).
 *
 * Conventions (all calls):
 *  - every floating-point array is fp64;
 *  - every pointer argument may be HOST or DEVICE memory (CUDA unified addressing decides);
 *    the library copies in/out synchronously on the context's stream and keeps no
 *    reference to caller memory after the call returns; the caller owns all its buffers;
 *  - fields are SoA [3][N3][N2][N1] = [component][z][y][x], x fastest (N1 = N2 = N3 = N for
 *    ib_create); p is [N3][N2][N1];
 *  - positions and nodal forces are AoS [np][3]; positions are unwrapped (indices mod N);
 *  - one ctx = one state = one CUDA stream; calls on one ctx must be externally
 *    serialised; the library owns all device memory of a ctx;
 *  - return codes: IB_OK (0) or a negative IB_E*; ib_last_error() gives a thread-local
 *    message for the last failing call.
 */
#ifndef IB_B200_H
#define IB_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ib_ctx ib_ctx;

enum {
  IB_OK = 0,
  IB_EINVAL = -1,       /* bad argument (shape, range, NULL, non-finite input)            */
  IB_ENOMEM = -2,       /* device allocation failed                                       */
  IB_ECUDA = -3,        /* CUDA runtime error (message in ib_last_error)                  */
  IB_ENONFINITE = -4,   /* a non-finite u or X appeared during ib_step                     */
  IB_ESTATE = -5,       /* call not valid in the current state (e.g. no structure set)    */
  IB_EDEGENERATE = -6   /* a link of zero length at rest                                 */
};

/* Patch flags: link families present in a structured patch (PAPER.md Q lattice, 697-710). */
enum {
  IB_WRAP1 = 1, IB_WRAP2 = 2,              /* i1 / i2 direction periodic                  */
  IB_STRETCH1 = 4, IB_STRETCH2 = 8,        /* (i1,i2)-(i1+1,i2) and (i1,i2)-(i1,i2+1)      */
  IB_BEND1 = 16, IB_BEND2 = 32,            /* (i1,i2)-(i1+2,i2) and (i1,i2)-(i1,i2+2)      */
  IB_TETHER = 64                           /* point tied to an anchor Y with stiffness kt */
};

/* One structured Lagrangian patch.  Point (i1,i2) is global index first + i2*n1 + i1.
 * Its block in stiffness[] starts at param_off (in doubles) and holds, in this order:
 * for each link family present (STRETCH1, STRETCH2, BEND1, BEND2): k[n1*n2] then
 * L0[n1*n2], indexed by the link's lower-index endpoint (i1,i2); for IB_TETHER:
 * kt[n1*n2] then Y[n1*n2*3].  A spring adds k(|d| - L0) d/|d| (d = X_j - X_i) to point i,
 * a tether adds kt (Y_i - X_i).  Forces are nodal (f * dq folded in; spread uses them as
 * F = sum F_node delta_h, reading Z12). */
typedef struct {
  int64_t first;
  int32_t n1, n2;
  uint32_t flags;
  uint32_t pad_;          /* must be 0 */
  int64_t param_off;
} ib_patch;

/* Options for ib_set_option. */
enum {
  IB_OPT_PRESSURE = 1,      /* 1: the last step of every ib_step batch also produces p   */
  IB_OPT_STAGE_TIMING = 2,  /* 1: record per-stage CUDA events inside ib_step            */
  IB_OPT_GRAPH = 3          /* 1 (default): run steps as a captured CUDA graph           */
};

/* Create a context for an N^3 periodic lattice of mesh width h (domain [0, N h)^3), fluid
 * density rho, viscosity mu, time step dt (PAPER.md 519-523, 602-605, 632-633).
 * Rejects: N not a power of two or N < 8 or N > 512; h <= 0; rho <= 0; mu < 0; dt <= 0.
 * The fluid starts at rest, no structure, step counter n = 0.  NULL on error. */
ib_ctx *ib_create(int32_t N, double h, double rho, double mu, double dt);
/* The same on an anisotropic N1 x N2 x N3 lattice (x, y, z) of mesh width h, domain
 * [0, N1 h) x [0, N2 h) x [0, N3 h) — e.g. the paper's 256 x 256 x 128 half-cube model
 * (PAPER.md 1003-1007).  Fields are then [3][N3][N2][N1] (x fastest), p is [N3][N2][N1].
 * Rejects, besides the ib_create cases per axis: N2 not a multiple of the x-pass row
 * block (32 / max(1, N1/32), at most N1: 4 for N1 = 256, 2 for 512). */
ib_ctx *ib_create3(int32_t N1, int32_t N2, int32_t N3, double h, double rho, double mu,
                   double dt);
void ib_destroy(ib_ctx *ctx);

/* Run all work of ctx on this CUDA stream (a cudaStream_t, e.g. torch's current stream);
 * NULL selects the library's own stream. */
int ib_set_stream(ib_ctx *ctx, void *cuda_stream);
int ib_set_option(ib_ctx *ctx, int32_t option, int64_t value);

/* Lagrangian structure: np points [np][3]; npatch patches covering points [0, np) with
 * stiffness[nstiff] as described above.  Rejects non-finite or out-of-range data and
 * (IB_EDEGENERATE) a link whose endpoints coincide at the given positions. */
int ib_set_structure(ib_ctx *ctx, const double *points, int64_t np, const ib_patch *patches,
                     int32_t npatch, const double *stiffness, int64_t nstiff);
/* Replace positions only ([np][3], same np as the structure): X^n of PAPER.md 602-605
 * (the boundary configuration the next step starts from).  Rejects non-finite values. */
int ib_set_positions(ib_ctx *ctx, const double *points);
/* Fluid velocity u^n on the lattice (PAPER.md 602-605, 632-633), [3][N3][N2][N1], x fastest.
 * Rejects non-finite values (IB_EINVAL).  Invalidates a pending pressure. */
int ib_set_velocity(ib_ctx *ctx, const double *u);
/* External drive (PAPER.md 988-993): F_idx[d] += amp * sin(2 pi n / period) * dir[d] at
 * step n (t^n = n dt).  dir == NULL: surface-normal drive ("orthogonal to the surface of
 * the window") — dir[d] is the unit normal t1 x t2 / |t1 x t2| of point idx[d]'s patch at
 * X^n, with tangents t1, t2 the central differences along i1, i2 (one-sided at an open
 * patch edge, periodic with IB_WRAP1/2); such points need a patch with n1, n2 >= 2.
 * n = 0 clears the drive.  ib_set_structure clears it. */
int ib_set_drive(ib_ctx *ctx, const int64_t *idx, int64_t n, const double *dir,
                 double amp_per_point, int32_t period_steps);
/* Fixed points (window plates, PAPER.md 914-922: "a rectangular grid, all of whose points
 * outside a given circle are fixed"): mask[np], mask[q] != 0 -> X(q) never moves; the point
 * still exerts its link forces on the fluid.  NULL clears; ib_set_structure clears it. */
int ib_set_fixed(ib_ctx *ctx, const uint8_t *mask);

/* Advance nsteps time steps of PAPER.md 608-628 (force, spread, eq:discreteNS1-2, then
 * eq:discreteX with u^{n+1} at X^n); n -> n + nsteps.  Synchronises the stream at the end.
 * Returns IB_ENONFINITE if u or X became non-finite: ib_last_error names the first bad
 * step; the batch has still run to its end on the device, so u, X and ib_get_step() are
 * at n + nsteps (the state is garbage from the bad step on; reset it before resuming). */
int ib_step(ib_ctx *ctx, int32_t nsteps);

/* Copy out u^n ([3][V], V = N1 N2 N3, may be NULL) and p^n ([V], may be NULL; needs
 * IB_OPT_PRESSURE enabled before the last ib_step, else IB_ESTATE): the velocity and
 * pressure of eq:discreteNS1-2 (PAPER.md 659-675) after the last step; p is the projection's
 * pressure with its null modes set to 0 (reading Z6). */
int ib_get_fields(ib_ctx *ctx, double *u, double *p);
/* Copy out X^n ([np][3], unwrapped) — the boundary positions of eq:discreteX (725-734). */
int ib_get_positions(ib_ctx *ctx, double *X);
/* Re-bin the points by lattice cell now (asynchronous on the ctx stream).  The binning is a
 * visiting order for spread and interpolation only (DESIGN.md §5 "cell binning"); ib_step
 * refreshes it every 32 steps by itself.  Exposed so that its cost can be timed. */
int ib_rebin(ib_ctx *ctx);
int64_t ib_get_step(ib_ctx *ctx);
int ib_set_step(ib_ctx *ctx, int64_t n);
int64_t ib_num_points(ib_ctx *ctx);

/* Per-stage device time (ms) accumulated since the last reset while IB_OPT_STAGE_TIMING
 * is on.  names: NUL-separated stage names written to names_buf (may be NULL).  Returns
 * the number of stages (<= cap). reset != 0 zeroes the accumulators afterwards. */
int ib_stage_times(ib_ctx *ctx, double *ms, int32_t cap, char *names_buf, int32_t names_cap,
                   int32_t reset);
/* Number of library kernel launches issued since the last reset (reset != 0 zeroes). */
int64_t ib_launch_count(ib_ctx *ctx, int32_t reset);

const char *ib_last_error(void);

/* ---- slab decomposition along z ----------
 * The paper partitions its fluid and material grids over processors (PAPER.md 801-807) and
 * needs it for the 2x refined model (1238-1245).  Rank `rank` of P owns the lattice planes
 * z in [rank L, (rank + 1) L), L = N3 / P; positions X are replicated on every rank.  One
 * step = ib_slab_phase 0, 1, 2, 3, 4 with the caller's exchange between phases (all
 * asynchronous on the ctx stream; the caller orders its collectives or copies on the same
 * stream):
 *   after 0: for each component c: all-to-all of s2[c] ([P dst][Ky][L][Pc] complex) into
 *            z[c] ([P src][Ky][L][Pc]), Ky = N2 / P, Pc = N1/2 + 2 (equal splits);
 *   after 1: the reverse all-to-all, z[c] -> s2[c];
 *   after 2: all-gather of edge_send ([3 planes][3][N2][N1] doubles: last, first, second
 *            owned plane) into edge_recv ([P][3][3][N2][N1]);
 *   after 3: all-gather of count_send (1 uint64) into count_recv ([P]) and of pack_send
 *            ([pack_cap] records (x, y, z, index) of doubles) into pack_recv ([P][pack_cap]).
 * Every buffer is caller-owned DEVICE memory that must outlive the ctx's use of it;
 * pack_cap >= np.  Requires N1, N2, N3 powers of two in [64, 512], P a power of two
 * dividing N2 and N3, L >= 8.  The other calls act on the slab: ib_set_structure,
 * ib_set_drive, ib_set_fixed, ib_set_positions take the whole (replicated) structure;
 * ib_set_velocity takes the WHOLE lattice u [3][N3][N2][N1]; ib_get_fields returns the owned
 * planes [3][L][N2][N1] (no pressure); ib_step and the ib_debug_* calls return IB_ESTATE. */
ib_ctx *ib_slab_create(int32_t N1, int32_t N2, int32_t N3, double h, double rho, double mu,
                       double dt, int32_t P, int32_t rank);
/* info[0..7] = P, rank, L, Ky, N1, N2, N3, Pc. */
int ib_slab_info(ib_ctx *ctx, int32_t *info, int32_t cap);
int ib_slab_set_buffers(ib_ctx *ctx, void *s2, void *z, double *edge_send, double *edge_recv,
                        void *pack_send, void *pack_recv, uint64_t *count_send,
                        uint64_t *count_recv, int64_t pack_cap);
/* Fused transposes: with P > 0, s2_peers[d] and z_peers[d] are rank d's s2
 * and z buffers (device pointers valid in this process: the other contexts of one process,
 * or peer / IPC-mapped memory of other GPUs), same shapes as this rank's.  Phase 0 then
 * stores the y-forward blocks bound for rank d straight into z_peers[d][.][rank] and phase 1
 * the z-solved blocks of source rank d straight into s2_peers[d][.][rank], so the caller
 * skips the exchanges after phases 0 and 1 and only orders the ranks (every rank's phase 0
 * before any rank's phase 1, every phase 1 before any phase 2).  P = 0 (arrays may be NULL)
 * returns to the exchange mode.  P must equal the slab count; after ib_slab_set_buffers. */
int ib_slab_set_peers(ib_ctx *ctx, int32_t P, void *const *s2_peers, void *const *z_peers);
/* Enqueue phase 0..4 of the next step (see above); phase 4 advances ib_get_step.  Phases
 * must come in order 0, 1, 2, 3, 4, 0, ... (IB_ESTATE otherwise). */
int ib_slab_phase(ib_ctx *ctx, int32_t phase);
/* Synchronise the ctx stream; IB_ENONFINITE (first bad step in ib_last_error) if u or X of
 * this rank became non-finite since the last call. */
int ib_slab_sync(ib_ctx *ctx);

/* ---- test-only entry points (same library; not part of the product contract) ----------
 * Each runs ONE stage of the step on the given inputs with the same kernels ib_step uses. */
int ib_debug_force(ib_ctx *ctx, double *f_out);                         /* [np][3], step n  */
int ib_debug_spread(ib_ctx *ctx, const double *f_node, double *F_out);   /* [np][3]->[3][V]  */
int ib_debug_interp(ib_ctx *ctx, const double *u, double *U_out);        /* [3][V]->[np][3]  */
/* r = rho u/dt - rho sum_k u_k D_k^{+-} u + F  ([3][V] each) */
int ib_debug_rhs(ib_ctx *ctx, const double *u, const double *F, double *r_out);
/* u^{n+1}, p^{n+1} from (u^n, F^n): the fluid part of the step (p_out may be NULL). */
int ib_debug_fluid(ib_ctx *ctx, const double *u, const double *F, double *u_out,
                   double *p_out);
/* S3c alone: u^ = (r^ - s (s.r^)/|s|^2)/d and p^ = -i (s.r^)/|s|^2 per mode
 * (null modes: u^ = r^/d, p^ = 0) from r^; half spectra as interleaved complex,
 * rhat/uhat [3][N3][N2][N1/2+1], phat [N3][N2][N1/2+1] (may be NULL).  Runs the product z
 * kernel between an inverse and a forward z transform.  IB_ESTATE unless N3 in [64, 512]. */
int ib_debug_project(ib_ctx *ctx, const double *rhat, double *uhat, double *phat);
/* Forward 3-D real-to-complex DFT of a real field [V] (unnormalised, e^{-2 pi i sum k_a j_a/N_a}):
 * out = complex half spectrum [N3][N2][N1/2+1] as interleaved (re, im). */
int ib_debug_fft(ib_ctx *ctx, const double *in, double *out);
/* Unnormalised inverse 3-D DFT (S3d) of a half spectrum [N3][N2][N1/2+1] (interleaved
 * re, im; the Hermitian half of a real field's spectrum) -> real field [V], through the
 * product inverse passes.  IB_ESTATE unless N3 in [64, 512]. */
int ib_debug_ifft(ib_ctx *ctx, const double *in, double *out);

#ifdef __cplusplus
}
#endif
#endif
