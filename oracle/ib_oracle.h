/* ib_oracle.h — the CPU oracle of the immersed-boundary time step (TEST INFRASTRUCTURE).
 *
 * Plain, slow, fp64 C written from PAPER.md §3.2 (lines 592-761).  It shares no code,
 * header, table or helper with the CUDA product path (include/ib.h,
 * paper_math_0301321_b200/csrc); only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.
 *
 * Layouts: fields are [c][z][y][x] (x fastest) on an N1 x N2 x N3 lattice (x, y, z),
 * x = h*(i,j,k), periodic; positions / nodal forces are [np][3].
 * Structures are structured patches: point (i1,i2) of patch p is
 * first[p] + i2*n1[p] + i1; stiffness block layout as documented in gen/configs.py.
 */
#ifndef IB_ORACLE_H
#define IB_ORACLE_H
#include <stdint.h>

#define IBO_WRAP1 1
#define IBO_WRAP2 2
#define IBO_STRETCH1 4
#define IBO_STRETCH2 8
#define IBO_BEND1 16
#define IBO_BEND2 32
#define IBO_TETHER 64

#ifdef __cplusplus
extern "C" {
#endif

void   ibo_set_threads(int nthreads);
int    ibo_get_threads(void);

/* Peskin 4-point phi(r), PAPER.md lines 745-759 (written exactly as the paper states). */
double ibo_phi(double r);

/* Step 1 — nodal Lagrangian force f^n: springs, tethers, drive.
 * drive_dir == NULL: surface-normal drive (PAPER.md 988-993) — each driven point is pushed
 * along the unit normal of its patch at X^n (central-difference tangents). */
void ibo_force(const double *X, int64_t np, int32_t npatch, const int64_t *first,
               const int32_t *n1, const int32_t *n2, const uint32_t *flags,
               const int64_t *param_off, const double *stiff,
               int64_t nd, const int64_t *drive_idx, const double *drive_dir,
               double drive_amp, int32_t drive_period, int64_t step, double *Fnode);

/* Step 2 — eq:discreteF: F = sum_q Fnode(q) delta_h(x - X(q)).
 * F[3][N^3] is overwritten.  Serial, point-index order. */
void ibo_spread(int32_t N1, int32_t N2, int32_t N3, double h, const double *X,
                const double *Fnode, int64_t np, double *F);

/* eq:discreteX interpolation: U(q) = sum_x u(x) delta_h(x-X(q)) h^3. */
void ibo_interp(int32_t N1, int32_t N2, int32_t N3, double h, const double *u, const double *X,
                int64_t np, double *U);

/* sum_k u_k^n D_k^{+-} u^n with the upwind rule of PAPER.md lines 676-691
 * (u_k = 0 -> backward difference, reading Z5).  adv[3][N^3]. */
void ibo_advect(int32_t N1, int32_t N2, int32_t N3, double h, const double *u, double *adv);

/* Right-hand side of eq:discreteNS1 after moving u^{n+1}-free terms right:
 * r = rho u^n / dt - rho sum_k u_k D_k^{+-} u^n + F^n. */
void ibo_rhs(int32_t N1, int32_t N2, int32_t N3, double h, double rho, double dt,
             const double *u, const double *F, double *r);

/* Unnormalised in-place 3-D complex DFT by radix-2 FFT along x, y, z ([N3][N2][N1] arrays).
 * sign = -1: X(k) = sum_j x(j) e^{-2 pi i sum_a k_a j_a / N_a}; sign = +1: the conjugate. */
void ibo_fft3(int32_t N1, int32_t N2, int32_t N3, double *re, double *im, int sign);

/* Solve eq:discreteNS1-2 for (u^{n+1}, p^{n+1}) given r.
 * u_out[3][N^3]; p_out[N^3] may be NULL. */
void ibo_solve(int32_t N1, int32_t N2, int32_t N3, double h, double rho, double mu, double dt,
               const double *r, double *u_out, double *p_out);

/* Step 3: rhs + solve. */
void ibo_fluid_step(int32_t N1, int32_t N2, int32_t N3, double h, double rho, double mu,
                    double dt, const double *u, const double *F, double *u_out, double *p_out);

/* nsteps full IB steps.  u[3][V] and X[np][3] in/out; p (may be
 * NULL) receives p^{n+1}: of the last step ([V]) when p_every == 0, of every step
 * ([nsteps][V]) when p_every != 0.  fixed (may be NULL): points with fixed[q] != 0 never
 * move but still exert their force (window plates, PAPER.md 914-922).  Returns 0, or 1 +
 * the 0-based step index at which a non-finite value appeared. */
int ibo_step(int32_t N1, int32_t N2, int32_t N3, double h, double rho, double mu, double dt,
             double *u, double *p, double *X, int64_t np, int32_t npatch, const int64_t *first,
             const int32_t *n1, const int32_t *n2, const uint32_t *flags,
             const int64_t *param_off, const double *stiff, int64_t nd,
             const int64_t *drive_idx, const double *drive_dir, double drive_amp,
             int32_t drive_period, int64_t step0, int32_t nsteps, int32_t p_every,
             const uint8_t *fixed);

#ifdef __cplusplus
}
#endif
#endif
