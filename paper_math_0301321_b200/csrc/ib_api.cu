// ib_api.cu — the C-ABI of include/ib.h: context, validation, memory, the step loop.
//
// One ib_step step is 7-9 launches on the context stream:
//   force+spread [+drive spread] -> xfwd (rhs + R2C-x) -> y fwd -> z fwd+solve+inv
//   -> y inv -> xinv (C2R-x, u^{n+1}) -> interp+update (X^{n+1}) -> step counter + 1.
// The step index lives in device memory, so one step is captured once as a CUDA graph and
// replayed (IB_OPT_GRAPH, default on); the points are re-binned by cell (5 launches) outside
// the graph every SORT_PERIOD steps.
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "api.cuh"

using namespace ibk;

static thread_local std::string g_err;

namespace ibk {

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

__global__ void k_count_nonfinite(const double *a, size_t n, unsigned long long *cnt) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  unsigned long long c = 0;
  for (; i < n; i += stride) c += !isfinite(a[i]);
  if (c) atomicAdd(cnt, c);
}


int count_nonfinite(ib_ctx *c, const double *d, size_t n, unsigned long long *out) {
  unsigned long long *cnt;
  CK(cudaMalloc(&cnt, sizeof(*cnt)));
  cudaMemsetAsync(cnt, 0, sizeof(*cnt), c->stream);
  k_count_nonfinite<<<592, 256, 0, c->stream>>>(d, n, cnt);
  c->launches++;
  cudaError_t e = cudaMemcpyAsync(out, cnt, sizeof(*cnt), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(cnt);
  CK(e);
  return IB_OK;
}

StructDev struct_dev(const ib_ctx *c) {
  StructDev s;
  s.X = c->X; s.np = c->np; s.perm = c->since_bin >= 0 ? c->perm : nullptr;
  s.Xs = c->since_bin >= 0 ? c->Xs : nullptr; s.patches = c->patches; s.npatch = c->npatch; s.stiff = c->stiff;
  s.nd = c->nd; s.drive_idx = c->drive_idx; s.drive_dir = c->drive_dir;
  s.drive_amp = c->drive_amp; s.drive_period = c->drive_period;
  return s;
}

void free_graph(ib_ctx *c) {
  if (c->graph) cudaGraphExecDestroy(c->graph);
  if (c->graph_chunk) cudaGraphExecDestroy(c->graph_chunk);
  c->graph = nullptr;
  c->graph_chunk = nullptr;
  c->graph_key = -1;
}

Sym sym_of(const ib_ctx *c) {
  return Sym{c->sym_s[0], c->sym_l[0], c->sym_s[1], c->sym_l[1], c->sym_s[2], c->sym_l[2]};
}

// The three strided spectrum passes: TMA column kernels when available (pencil length in
// [64, 512]), else the cp.async pencil kernels.
cudaError_t yfwd(ib_ctx *c, cudaStream_t s) {
  if (c->maps.y_ok) return launch_colfft(c->g, 1, c->maps, nullptr, c->tw[1], sym_of(c), s);
  return launch_ypass(c->g, -1, c->spec, 1, c->spec2, 2, 3, c->tw[1], s);
}
cudaError_t zsolve(ib_ctx *c, double2 *pspec, cudaStream_t s) {
  if (c->maps.z_ok) return launch_colfft(c->g, 0, c->maps, pspec, c->tw[2], sym_of(c), s);
  return launch_zpass(c->g, 0, c->spec2, pspec, c->tw[2], sym_of(c), s);
}
cudaError_t yinv(ib_ctx *c, cudaStream_t s) {
  if (c->maps.y_ok) return launch_colfft(c->g, 2, c->maps, nullptr, c->tw[1], sym_of(c), s);
  return launch_ypass(c->g, +1, c->spec2, 2, c->spec, 1, 3, c->tw[1], s);
}

// Pressure half-spectrum p^ written by the z solve (S2 layout) -> p [V] real.  With the
// TMA z pass p^ is in full (ky, kz, kx) order and ps must hold 3 component slots (the
// inverse-z column pass transforms all three; slots 1-2 are scratch).
cudaError_t pressure_to_real(ib_ctx *c, double2 *ps, double2 *ps1, double *out, cudaStream_t s) {
  cudaError_t e;
  if (c->maps.z_ok) {
    TmaMaps m;
    if (!colfft_encode_s2(c->g, ps, &m.s2_2d)) return cudaErrorInvalidValue;
    m.z_ok = true;
    if ((e = launch_colfft(c->g, 4, m, nullptr, c->tw[2], sym_of(c), s)) != cudaSuccess) return e;
  }
  if ((e = launch_ypass(c->g, +1, ps, 2, ps1, 1, 1, c->tw[1], s)) != cudaSuccess) return e;
  return launch_xinv(c->g, ps1, out, 1, c->tw[0], c->twM, nullptr, nullptr, 0, s);
}

size_t spec1_elems(const ib_ctx *c) { return (size_t)c->g.N2 * c->g.N3 * c->g.P; }
size_t pspec_elems(const ib_ctx *c) { return (size_t)(c->maps.z_ok ? 3 : 1) * spec1_elems(c); }

// x passes: the forward pass is fluid.cu's k_xfwd; the inverse uses the TMA kernel when
// available (N in [64, 256]).
cudaError_t xfwd(ib_ctx *c, int mode, const double *u, double *F, unsigned *rowflag,
                 double *r_out, cudaStream_t s) {
  if (mode == 2)
    return launch_xfwd(c->g, 2, nullptr, nullptr, nullptr, u, nullptr, c->spec, c->tw[0], c->twM,
                       nullptr, s);
  XMapsU tmp;
  const XMapsU *um = &c->umaps;
  if (u != c->u) {                      // debug arrays: maps encoded on the fly
    xfwd_encode_u(c->g, u, &tmp);
    um = &tmp;
  }
  return launch_xfwd(c->g, mode, u, F, rowflag, nullptr, r_out, c->spec, c->tw[0], c->twM, um, s);
}
cudaError_t xinv(ib_ctx *c, double *out, const long long *dev_n, long long n, long long *flag,
                 cudaStream_t s) {
  if (c->xok) return launch_xinv_tma(c->g, c->smaps, out, c->tw[0], c->twM, flag, dev_n, n, s);
  return launch_xinv(c->g, c->spec, out, 3, c->tw[0], c->twM, flag, dev_n, n, s);
}

// (Re)bin the points by base cell when the permutation is missing or SORT_PERIOD steps old.
cudaError_t ensure_binned(ib_ctx *c, cudaStream_t s) {
  if (c->np == 0 || (c->since_bin >= 0 && c->since_bin < SORT_PERIOD)) return cudaSuccess;
  cudaError_t e = launch_bin(c->g, c->X, c->np, c->bincnt, c->binsum, c->perm, c->Xs, s);
  if (e == cudaSuccess) {
    c->since_bin = 0;
    c->launches += 6;
  }
  return e;
}

// Enqueue one step (binning is the caller's job).  The step index is read on the device
// from c->dev_n and advanced by the step's last launch, so the same sequence is captured once
// as a CUDA graph and replayed.
cudaError_t enqueue_step(ib_ctx *c, bool pressure, cudaEvent_t *ev) {
  const FluidGeom &g = c->g;
  cudaStream_t s = c->stream;
  const long long *dev_n = c->dev_n, n = 0;
  cudaError_t e;
  StructDev sd = struct_dev(c);
  auto mark = [&](int k) { if (ev) cudaEventRecord(ev[k], s); };
  mark(0);
  if ((e = launch_force_spread(sd, g, nullptr, dev_n, n, c->F, c->rowflag, s)) != cudaSuccess) return e;
  mark(1);
  if ((e = xfwd(c, 0, c->u, c->F, c->rowflag, nullptr, s)) != cudaSuccess) return e;
  mark(2);
  if ((e = yfwd(c, s)) != cudaSuccess) return e;
  mark(3);
  if ((e = zsolve(c, pressure ? c->pspec : nullptr, s)) != cudaSuccess) return e;
  mark(4);
  if ((e = yinv(c, s)) != cudaSuccess) return e;
  mark(5);
  if ((e = xinv(c, c->u, dev_n, n, c->flag, s)) != cudaSuccess) return e;
  mark(6);
  if ((e = launch_interp(g, c->u, c->X, c->np, nullptr, c->flag, dev_n, n, sd.perm, c->fixed, s,
                         nullptr, nullptr, c->Xs)) != cudaSuccess) return e;
  mark(7);
  return launch_step_inc(c->dev_n, s);
}

// x forward, y forward, z solve, y inverse, x inverse, step counter; force + spread (drive
// included) and interp with points
int64_t launches_per_step(const ib_ctx *c, bool pressure) {
  (void)pressure;
  return 6 + (c->np > 0 ? 2 : 0);
}

// m = 1 or GRAPH_CHUNK consecutive steps as a CUDA graph (captured on first use, replayed
// until invalidated).  The chunk graph saves the graph-to-graph launch gap of the steps
// inside it; ib_step uses it when no re-binning falls inside the chunk.
cudaError_t graph_steps(ib_ctx *c, int m) {
  cudaGraphExec_t &ge = m == 1 ? c->graph : c->graph_chunk;
  if (!ge) {
    cudaGraph_t gr = nullptr;
    cudaError_t e = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return e;
    for (int k = 0; k < m && e == cudaSuccess; ++k) e = enqueue_step(c, false, nullptr);
    cudaError_t e2 = cudaStreamEndCapture(c->stream, &gr);
    if (e == cudaSuccess) e = e2;
    if (e == cudaSuccess) e = cudaGraphInstantiate(&ge, gr, 0);
    if (gr) cudaGraphDestroy(gr);
    if (e != cudaSuccess) { ge = nullptr; return e; }
  }
  return cudaGraphLaunch(ge, c->stream);
}

struct Tmp {
  std::vector<void *> ptrs;
  ~Tmp() { for (void *p : ptrs) cudaFree(p); }
  template <class T> cudaError_t get(T **p, size_t n) {
    cudaError_t e = dalloc(p, n);
    if (e == cudaSuccess) ptrs.push_back(*p);
    return e;
  }
};

}  // namespace ibk

extern "C" {

const char *ib_last_error(void) { return g_err.c_str(); }

static bool pow2_in(int32_t n, int32_t lo, int32_t hi) { return n >= lo && n <= hi && !(n & (n - 1)); }

// rows per x-pass tile for a row length N1: the y extent N2 must be a multiple of the
// forward pass's (fluid.cu XCfg) and of the TMA inverse pass's (xpass_tma.cu XT) row block
static int32_t x_rows(int32_t N1) {
  const int32_t a = xfwd_rows(N1);
  const int32_t M = N1 / 2, T = M >= 16 ? M / 16 : 1, b = 32 / T < N1 ? 32 / T : N1;
  return a > b ? a : b;
}

ib_ctx *ib_create3(int32_t N1, int32_t N2, int32_t N3, double h, double rho, double mu,
                   double dt) {
  if (!pow2_in(N1, 8, 512) || !pow2_in(N2, 8, 512) || !pow2_in(N3, 8, 512)) {
    fail(IB_EINVAL, "N1, N2, N3 must be powers of two in [8, 512]");
    return nullptr;
  }
  if (N2 % x_rows(N1)) {
    fail(IB_EINVAL, "N2 must be a multiple of " + std::to_string(x_rows(N1)) + " for N1 = " +
                        std::to_string(N1));
    return nullptr;
  }
  if (!(h > 0) || !std::isfinite(h)) { fail(IB_EINVAL, "h must be > 0"); return nullptr; }
  if (!(rho > 0) || !std::isfinite(rho)) { fail(IB_EINVAL, "rho must be > 0"); return nullptr; }
  if (!(mu >= 0) || !std::isfinite(mu)) { fail(IB_EINVAL, "mu must be >= 0"); return nullptr; }
  if (!(dt > 0) || !std::isfinite(dt)) { fail(IB_EINVAL, "dt must be > 0"); return nullptr; }
  ib_ctx *c = new ib_ctx();
  c->g.N1 = N1; c->g.N2 = N2; c->g.N3 = N3;
  c->g.M = N1 / 2; c->g.P = N1 / 2 + 2;
  c->g.V = (int64_t)N1 * N2 * N3;
  c->g.h = h; c->g.invh = 1.0 / h; c->g.rho = rho; c->g.mu = mu; c->g.dt = dt;
  geom_whole(c->g);
  auto bad = [&](cudaError_t e, const char *what) {
    fail(e == cudaErrorMemoryAllocation ? IB_ENOMEM : IB_ECUDA,
         std::string("ib_create: ") + what + ": " + cudaGetErrorString(e));
    ib_destroy(c);
    return (ib_ctx *)nullptr;
  };
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking)) != cudaSuccess) return bad(e, "stream");
  c->stream = c->own_stream;
  const size_t V = (size_t)c->g.V;
  const size_t S = (size_t)3 * spec1_elems(c);
  if ((e = dalloc(&c->u, 3 * V)) != cudaSuccess) return bad(e, "u");
  if ((e = dalloc(&c->F, 3 * V)) != cudaSuccess) return bad(e, "F");
  if ((e = dalloc(&c->spec, S)) != cudaSuccess) return bad(e, "spectrum");
  if ((e = dalloc(&c->spec2, S)) != cudaSuccess) return bad(e, "spectrum");
  if ((e = dalloc(&c->rowflag, (size_t)N2 * N3)) != cudaSuccess) return bad(e, "row flags");
  if ((e = cudaMemsetAsync(c->rowflag, 0, (size_t)N2 * N3 * sizeof(unsigned), c->stream)) != cudaSuccess) return bad(e, "memset");
  const int32_t L[3] = {N1, N2, N3};
  for (int a = 0; a < 3; ++a) {
    if ((e = dalloc(&c->tw[a], (size_t)L[a])) != cudaSuccess) return bad(e, "tables");
    if ((e = dalloc(&c->sym_s[a], (size_t)L[a])) != cudaSuccess) return bad(e, "tables");
    if ((e = dalloc(&c->sym_l[a], (size_t)L[a])) != cudaSuccess) return bad(e, "tables");
  }
  if ((e = dalloc(&c->twM, N1 / 2)) != cudaSuccess) return bad(e, "tables");
  if ((e = dalloc(&c->flag, 1)) != cudaSuccess) return bad(e, "flag");
  if ((e = dalloc(&c->dev_n, 1)) != cudaSuccess) return bad(e, "flag");
  if ((e = cudaMallocHost(&c->flag_h, sizeof(long long))) != cudaSuccess) return bad(e, "flag");
  for (int k = 0; k <= STAGE_COUNT; ++k)
    if ((e = cudaEventCreate(&c->ev[k])) != cudaSuccess) return bad(e, "events");
  if ((e = cudaMemsetAsync(c->u, 0, 3 * V * sizeof(double), c->stream)) != cudaSuccess) return bad(e, "memset");
  if ((e = cudaMemsetAsync(c->F, 0, 3 * V * sizeof(double), c->stream)) != cudaSuccess) return bad(e, "memset");
  for (int a = 0; a < 3; ++a)
    if ((e = fluid_setup_attributes(L[a])) != cudaSuccess) return bad(e, "attributes");
  if ((e = colfft_make_maps(c->g, c->spec, c->spec2, &c->maps)) != cudaSuccess) return bad(e, "TMA tensor maps");
#ifndef IBK_NO_XFTMA
  xfwd_encode_u(c->g, c->u, &c->umaps);   // !ok (cp.async tile copy) when N1 < 16
#endif
#ifndef IBK_NO_XTMA   // dev switch: the per-CTA row kernels of fluid.cu for comparison
  if (xpass_supported(N1)) {
    if (!xpass_encode_s1(c->g, c->spec, &c->smaps))
      return bad(cudaErrorInvalidValue, "TMA tensor maps (x passes)");
    c->xok = true;
  }
#endif
  if ((e = init_tables(c)) != cudaSuccess) return bad(e, "tables");
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return bad(e, "sync");
  return c;
}

ib_ctx *ib_create(int32_t N, double h, double rho, double mu, double dt) {
  return ib_create3(N, N, N, h, rho, mu, dt);
}

void ib_destroy(ib_ctx *c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  free_graph(c);
  dfree(c->u); dfree(c->F); dfree(c->rowflag); dfree(c->spec); dfree(c->spec2); dfree(c->pspec); dfree(c->pspec1); dfree(c->p);
  for (int a = 0; a < 3; ++a) { dfree(c->tw[a]); dfree(c->sym_s[a]); dfree(c->sym_l[a]); }
  dfree(c->twM);
  dfree(c->X); dfree(c->patches); dfree(c->stiff); dfree(c->drive_idx); dfree(c->drive_dir);
  dfree(c->perm); dfree(c->Xs); dfree(c->bincnt); dfree(c->binsum); dfree(c->fixed);
  dfree(c->flag); dfree(c->dev_n);
  if (c->flag_h) cudaFreeHost(c->flag_h);
  for (int k = 0; k <= STAGE_COUNT; ++k) if (c->ev[k]) cudaEventDestroy(c->ev[k]);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  delete c;
}

int ib_set_stream(ib_ctx *c, void *stream) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  CK(cudaStreamSynchronize(c->stream));
  c->stream = stream ? (cudaStream_t)stream : c->own_stream;
  free_graph(c);
  return IB_OK;
}

int ib_set_option(ib_ctx *c, int32_t opt, int64_t value) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  switch (opt) {
    case IB_OPT_PRESSURE:
      if (c->slab_P && value) return fail(IB_ESTATE, "slab context: no pressure output");
      c->want_p = value != 0;
      if (c->want_p && !c->pspec) {
        CK(dalloc(&c->pspec, pspec_elems(c)));
        CK(dalloc(&c->pspec1, spec1_elems(c)));
        CK(dalloc(&c->p, (size_t)c->g.V));
      }
      return IB_OK;
    case IB_OPT_STAGE_TIMING: c->timing = value != 0; return IB_OK;
    case IB_OPT_GRAPH: c->use_graph = value != 0; free_graph(c); return IB_OK;
    default: return fail(IB_EINVAL, "unknown option");
  }
}

int ib_set_structure(ib_ctx *c, const double *points, int64_t np, const ib_patch *patches,
                     int32_t npatch, const double *stiffness, int64_t nstiff) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  if (np < 0 || npatch < 0 || nstiff < 0) return fail(IB_EINVAL, "negative count");
  if ((np > 0 && (!points || !patches)) || (nstiff > 0 && !stiffness))
    return fail(IB_EINVAL, "NULL array with non-zero count");
  if (np > 0 && npatch == 0) return fail(IB_EINVAL, "points without patches");
  if (np >= (int64_t)1 << 31) return fail(IB_EINVAL, "too many points");
  std::vector<double> X, S;
  std::vector<ib_patch> P;
  CK(to_host(X, points, (size_t)np * 3, c->stream));
  CK(to_host(P, patches, (size_t)npatch, c->stream));
  CK(to_host(S, stiffness, (size_t)nstiff, c->stream));
  for (int64_t i = 0; i < 3 * np; ++i)
    if (!std::isfinite(X[i])) return fail(IB_EINVAL, "non-finite position at point " + std::to_string(i / 3));
  int64_t next = 0;
  for (int32_t p = 0; p < npatch; ++p) {
    const ib_patch &q = P[p];
    const std::string tag = "patch " + std::to_string(p) + ": ";
    if (q.first != next) return fail(IB_EINVAL, tag + "patches must tile [0, np) in order");
    if (q.n1 < 1 || q.n2 < 1) return fail(IB_EINVAL, tag + "n1, n2 must be >= 1");
    if (q.flags & ~127u) return fail(IB_EINVAL, tag + "unknown flag bits");
    if (q.pad_ != 0) return fail(IB_EINVAL, tag + "pad_ must be 0");
    const int64_t npts = (int64_t)q.n1 * q.n2;
    next += npts;
    int nfam = 0;
    for (int f = 0; f < 4; ++f) nfam += (q.flags >> (2 + f)) & 1;
    const int64_t need = 2 * nfam * npts + ((q.flags & IB_TETHER) ? 4 * npts : 0);
    if (q.param_off < 0 || q.param_off + need > nstiff) return fail(IB_EINVAL, tag + "stiffness block out of range");
    for (int64_t k = 0; k < need; ++k)
      if (!std::isfinite(S[q.param_off + k])) return fail(IB_EINVAL, tag + "non-finite stiffness at offset " + std::to_string(q.param_off + k));
    // zero-length links at the given positions
    int64_t b = q.param_off;
    for (int f = 0; f < 4; ++f) {
      if (!(q.flags & (IB_STRETCH1 << f))) continue;
      const bool ax1 = (f & 1) == 0;
      const int off = f < 2 ? 1 : 2;
      const int n = ax1 ? q.n1 : q.n2;
      const bool wrap = (q.flags & (ax1 ? IB_WRAP1 : IB_WRAP2)) != 0;
      for (int32_t i2 = 0; i2 < q.n2; ++i2)
        for (int32_t i1 = 0; i1 < q.n1; ++i1) {
          const int cidx = ax1 ? i1 : i2;
          if (!(cidx + off < n || wrap)) continue;
          const int cf = (cidx + off) % n;
          const int64_t li = (int64_t)i2 * q.n1 + i1;
          const int64_t lj = ax1 ? (int64_t)i2 * q.n1 + cf : (int64_t)cf * q.n1 + i1;
          const double *a = &X[3 * (q.first + li)], *bb = &X[3 * (q.first + lj)];
          if (a[0] == bb[0] && a[1] == bb[1] && a[2] == bb[2])
            return fail(IB_EDEGENERATE, tag + "zero-length link between points " +
                                            std::to_string(q.first + li) + " and " +
                                            std::to_string(q.first + lj));
        }
      b += 2 * (int64_t)q.n1 * q.n2;
    }
  }
  if (next != np) return fail(IB_EINVAL, "patches cover " + std::to_string(next) + " points, np = " + std::to_string(np));
  // upload
  free_graph(c);
  CK(cudaStreamSynchronize(c->stream));
  dfree(c->X); dfree(c->patches); dfree(c->stiff); dfree(c->perm); dfree(c->Xs);
  c->X = nullptr; c->patches = nullptr; c->stiff = nullptr; c->perm = nullptr; c->Xs = nullptr;
  c->since_bin = -1;
  CK(dalloc(&c->X, (size_t)np * 3));
  CK(dalloc(&c->perm, (size_t)np));
  CK(dalloc(&c->Xs, (size_t)np * 3));
  if (np > 0 && !c->bincnt) {
    CK(dalloc(&c->bincnt, (size_t)c->g.Vg));            // cells of the whole lattice
    CK(dalloc(&c->binsum, (size_t)bin_scan_blocks(c->g.Vg)));
  }
  CK(dalloc(&c->patches, (size_t)npatch));
  CK(dalloc(&c->stiff, (size_t)nstiff));
  CK(copy_sync(c->X, X.data(), X.size() * sizeof(double), c->stream));
  CK(copy_sync(c->patches, P.data(), P.size() * sizeof(ib_patch), c->stream));
  CK(copy_sync(c->stiff, S.data(), S.size() * sizeof(double), c->stream));
  c->np = np; c->npatch = npatch; c->nstiff = nstiff; c->patches_h = P;
  // a drive that no longer fits is dropped
  if (c->nd > 0) { dfree(c->drive_idx); dfree(c->drive_dir); c->drive_idx = nullptr; c->drive_dir = nullptr; c->nd = 0; }
  dfree(c->fixed);                       // a fixed mask belongs to the old structure
  c->fixed = nullptr;
  return IB_OK;
}

int ib_set_positions(ib_ctx *c, const double *points) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  if (c->np == 0) return IB_OK;
  if (!points) return fail(IB_EINVAL, "points is NULL");
  CK(copy_sync(c->X, points, (size_t)c->np * 3 * sizeof(double), c->stream));
  c->since_bin = -1;
  unsigned long long bad = 0;
  int rc = count_nonfinite(c, c->X, (size_t)c->np * 3, &bad);
  if (rc) return rc;
  if (bad) return fail(IB_EINVAL, "non-finite positions");
  return IB_OK;
}

int ib_set_velocity(ib_ctx *c, const double *u) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  if (!u) return fail(IB_EINVAL, "u is NULL");
  size_t nu = (size_t)3 * c->g.V;
  if (c->slab_P) {
    // slab: u is the WHOLE lattice [3][N3][N2][N1]; this rank keeps its planes and ghosts
    // (global planes z0 - 1 .. z0 + L + 1, periodic)
    const FluidGeom &g = c->g;
    const size_t plane = (size_t)g.N1 * g.N2, Vu = plane * g.uN3;
    for (int comp = 0; comp < 3; ++comp)
      for (int p = 0; p < g.uN3; ++p) {
        const int zg = ((g.z0 - g.uz0 + p) % g.N3g + g.N3g) % g.N3g;
        CK(cudaMemcpyAsync(c->u + comp * Vu + p * plane, u + comp * (size_t)g.Vg + zg * plane,
                           plane * sizeof(double), cudaMemcpyDefault, c->stream));
      }
    CK(cudaStreamSynchronize(c->stream));
    nu = 3 * Vu;
  } else {
    CK(copy_sync(c->u, u, nu * sizeof(double), c->stream));
  }
  unsigned long long bad = 0;
  int rc = count_nonfinite(c, c->u, nu, &bad);
  if (rc) return rc;
  if (bad) return fail(IB_EINVAL, "non-finite velocity");
  c->have_p = false;
  return IB_OK;
}

int ib_set_drive(ib_ctx *c, const int64_t *idx, int64_t n, const double *dir,
                 double amp_per_point, int32_t period_steps) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  if (n < 0) return fail(IB_EINVAL, "negative drive count");
  if (n > 0) {
    if (!idx) return fail(IB_EINVAL, "NULL drive indices");
    if (period_steps < 1) return fail(IB_EINVAL, "period_steps must be >= 1");
    if (!std::isfinite(amp_per_point)) return fail(IB_EINVAL, "non-finite amplitude");
    std::vector<int64_t> I;
    std::vector<double> D;
    CK(to_host(I, idx, (size_t)n, c->stream));
    if (dir) CK(to_host(D, dir, (size_t)n * 3, c->stream));
    for (int64_t d = 0; d < n; ++d) {
      if (I[d] < 0 || I[d] >= c->np) return fail(IB_EINVAL, "drive index out of range: " + std::to_string(I[d]));
      if (dir) {
        for (int k = 0; k < 3; ++k)
          if (!std::isfinite(D[3 * d + k])) return fail(IB_EINVAL, "non-finite drive direction");
      } else {                 // surface-normal drive: the point's patch must be a 2-D grid
        int32_t p = 0;
        while (p + 1 < c->npatch && c->patches_h[p + 1].first <= I[d]) ++p;
        if (c->patches_h[p].n1 < 2 || c->patches_h[p].n2 < 2)
          return fail(IB_EINVAL, "normal drive on point " + std::to_string(I[d]) +
                                     " of a patch with n1 or n2 < 2 (no surface normal)");
      }
    }
    free_graph(c);
    CK(cudaStreamSynchronize(c->stream));
    dfree(c->drive_idx); dfree(c->drive_dir);
    c->drive_idx = nullptr; c->drive_dir = nullptr;
    CK(dalloc(&c->drive_idx, (size_t)n));
    CK(copy_sync(c->drive_idx, I.data(), I.size() * sizeof(int64_t), c->stream));
    if (dir) {
      CK(dalloc(&c->drive_dir, (size_t)n * 3));
      CK(copy_sync(c->drive_dir, D.data(), D.size() * sizeof(double), c->stream));
    }
  } else {
    free_graph(c);
  }
  c->nd = n;
  c->drive_amp = amp_per_point;
  c->drive_period = n > 0 ? period_steps : 1;
  return IB_OK;
}

int ib_set_fixed(ib_ctx *c, const uint8_t *mask) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  free_graph(c);
  CK(cudaStreamSynchronize(c->stream));
  dfree(c->fixed);
  c->fixed = nullptr;
  if (mask && c->np > 0) {
    CK(dalloc(&c->fixed, (size_t)c->np));
    CK(copy_sync(c->fixed, mask, (size_t)c->np, c->stream));
  }
  return IB_OK;
}

int ib_step(ib_ctx *c, int32_t nsteps) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  if (c->slab_P) return fail(IB_ESTATE, "slab context: step with ib_slab_phase 0..4");
  if (nsteps < 0) return fail(IB_EINVAL, "nsteps < 0");
  if (nsteps == 0) return IB_OK;
  cudaStream_t s = c->stream;
  *c->flag_h = LLONG_MAX;
  CK(cudaMemcpyAsync(c->flag, c->flag_h, sizeof(long long), cudaMemcpyHostToDevice, s));
  const bool timing = c->timing;
  const size_t per = STAGE_COUNT + 1;
  if (timing) {
    while (c->ev_pool.size() < (size_t)nsteps * per) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      c->ev_pool.push_back(e);
    }
  }
  const long long n0 = c->n;
  CK(cudaMemcpyAsync(c->dev_n, &n0, sizeof(long long), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));                 // n0 lives on the host stack
  for (int32_t k = 0; k < nsteps;) {
    const bool pressure = c->want_p && k == nsteps - 1;
    CK(ensure_binned(c, s));                    // outside the graph (it holds only pointers)
    int32_t m = 1;
    if (c->use_graph && !timing && !pressure) {
      // GRAPH_CHUNK steps in one graph when neither the next re-binning (same schedule as
      // step by step: every SORT_PERIOD steps) nor the pressure step falls inside them
      const int32_t plain_left = nsteps - k - (c->want_p ? 1 : 0);
      const bool room = c->np == 0 || c->since_bin + GRAPH_CHUNK <= SORT_PERIOD;
      if (plain_left >= GRAPH_CHUNK && room) m = GRAPH_CHUNK;
      CK(graph_steps(c, m));
    } else {
      CK(enqueue_step(c, pressure, timing ? &c->ev_pool[k * per] : nullptr));
    }
    c->since_bin += m;
    c->launches += m * launches_per_step(c, pressure);
    k += m;
  }
  CK(cudaMemcpyAsync(c->flag_h, c->flag, sizeof(long long), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (timing) {
    for (int32_t k = 0; k < nsteps; ++k)
      for (int st = 0; st < STAGE_COUNT; ++st) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->ev_pool[k * per + st], c->ev_pool[k * per + st + 1]));
        c->stage_ms[st] += ms;
      }
  }
  const long long bad = *c->flag_h;
  c->have_p = c->want_p;
  if (bad != LLONG_MAX) {
    // the batch ran to its end on the device (u, X and the device counter are at n0 +
    // nsteps), so the host counter follows them; the first bad step is in the message
    c->n = n0 + nsteps;
    return fail(IB_ENONFINITE, "non-finite u or X first at step " + std::to_string(bad) +
                                   " (state left at step " + std::to_string(c->n) + ")");
  }
  c->n += nsteps;
  return IB_OK;
}

int ib_get_fields(ib_ctx *c, double *u, double *p) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  if (c->slab_P) {            // slab: the owned planes [3][L][N2][N1]; no pressure
    if (p) return fail(IB_ESTATE, "slab context: no pressure output");
    if (u) {
      const FluidGeom &g = c->g;
      const size_t plane = (size_t)g.N1 * g.N2, Vu = plane * g.uN3;
      for (int comp = 0; comp < 3; ++comp)
        CK(cudaMemcpyAsync(u + comp * (size_t)g.V, c->u + comp * Vu + g.uz0 * plane,
                           (size_t)g.V * sizeof(double), cudaMemcpyDefault, c->stream));
      CK(cudaStreamSynchronize(c->stream));
    }
    return IB_OK;
  }
  if (u) CK(copy_sync(u, c->u, (size_t)3 * c->g.V * sizeof(double), c->stream));
  if (p) {
    if (!c->have_p || !c->pspec) return fail(IB_ESTATE, "pressure not available: enable IB_OPT_PRESSURE before ib_step");
    CK(pressure_to_real(c, c->pspec, c->pspec1, c->p, c->stream));
    c->launches += c->maps.z_ok ? 3 : 2;
    CK(copy_sync(p, c->p, (size_t)c->g.V * sizeof(double), c->stream));
  }
  return IB_OK;
}

int ib_get_positions(ib_ctx *c, double *X) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  if (c->np == 0) return IB_OK;
  if (!X) return fail(IB_EINVAL, "X is NULL");
  CK(copy_sync(X, c->X, (size_t)c->np * 3 * sizeof(double), c->stream));
  return IB_OK;
}

int ib_rebin(ib_ctx *c) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  if (c->np == 0) return IB_OK;
  c->since_bin = -1;
  CK(ensure_binned(c, c->stream));
  return IB_OK;
}

int64_t ib_get_step(ib_ctx *c) { return c ? c->n : -1; }
int ib_set_step(ib_ctx *c, int64_t n) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  if (n < 0) return fail(IB_EINVAL, "n < 0");
  c->n = n;
  if (c->slab_P) {            // slab phases read the device counter directly
    const long long v = n;
    CK(copy_sync(c->dev_n, &v, sizeof(v), c->stream));
  }
  return IB_OK;
}
int64_t ib_num_points(ib_ctx *c) { return c ? c->np : -1; }

int ib_stage_times(ib_ctx *c, double *ms, int32_t cap, char *names, int32_t names_cap,
                   int32_t reset) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  static const char *nm[STAGE_COUNT] = {"force_spread", "xfwd_rhs_r2c", "y_fwd", "z_solve",
                                        "y_inv", "xinv_c2r", "interp_update"};
  const int n = cap < STAGE_COUNT ? cap : STAGE_COUNT;
  for (int k = 0; k < n; ++k) if (ms) ms[k] = c->stage_ms[k];
  if (names && names_cap > 0) {
    int pos = 0;
    for (int k = 0; k < n; ++k) {
      const int L = (int)strlen(nm[k]);
      if (pos + L + 1 > names_cap) break;
      memcpy(names + pos, nm[k], L + 1);
      pos += L + 1;
    }
  }
  if (reset) for (int k = 0; k < STAGE_COUNT; ++k) c->stage_ms[k] = 0.0;
  return n;
}

int64_t ib_launch_count(ib_ctx *c, int32_t reset) {
  if (!c) return -1;
  const int64_t v = c->launches;
  if (reset) c->launches = 0;
  return v;
}

// ------------------------------------------------------------------ debug entry points

int ib_debug_force(ib_ctx *c, double *f_out) {
  if (c && c->slab_P) return fail(IB_ESTATE, "debug entry points need a whole-lattice context");
  if (!c || !f_out) return fail(IB_EINVAL, "NULL argument");
  if (c->np == 0) return IB_OK;
  Tmp t; double *f;
  CK(t.get(&f, (size_t)c->np * 3));
  CK(launch_force(struct_dev(c), nullptr, c->n, f, c->stream));
  CK(copy_sync(f_out, f, (size_t)c->np * 3 * sizeof(double), c->stream));
  return IB_OK;
}

int ib_debug_spread(ib_ctx *c, const double *f_node, double *F_out) {
  if (c && c->slab_P) return fail(IB_ESTATE, "debug entry points need a whole-lattice context");
  if (!c || !f_node || !F_out) return fail(IB_EINVAL, "NULL argument");
  Tmp t; double *f, *F;
  const size_t V = (size_t)c->g.V;
  CK(t.get(&F, 3 * V));
  CK(cudaMemsetAsync(F, 0, 3 * V * sizeof(double), c->stream));
  if (c->np > 0) {
    CK(t.get(&f, (size_t)c->np * 3));
    CK(copy_sync(f, f_node, (size_t)c->np * 3 * sizeof(double), c->stream));
    CK(ensure_binned(c, c->stream));
    CK(launch_force_spread(struct_dev(c), c->g, f, nullptr, c->n, F, nullptr, c->stream));
  }
  CK(copy_sync(F_out, F, 3 * V * sizeof(double), c->stream));
  return IB_OK;
}

int ib_debug_interp(ib_ctx *c, const double *u, double *U_out) {
  if (c && c->slab_P) return fail(IB_ESTATE, "debug entry points need a whole-lattice context");
  if (!c || !u || !U_out) return fail(IB_EINVAL, "NULL argument");
  if (c->np == 0) return IB_OK;
  Tmp t; double *ud, *U;
  const size_t V = (size_t)c->g.V;
  CK(t.get(&ud, 3 * V));
  CK(t.get(&U, (size_t)c->np * 3));
  CK(copy_sync(ud, u, 3 * V * sizeof(double), c->stream));
  CK(ensure_binned(c, c->stream));
  const StructDev sd = struct_dev(c);
  CK(launch_interp(c->g, ud, c->X, c->np, U, nullptr, nullptr, 0, sd.perm, nullptr, c->stream,
                   nullptr, nullptr, c->Xs));
  CK(copy_sync(U_out, U, (size_t)c->np * 3 * sizeof(double), c->stream));
  return IB_OK;
}

int ib_debug_rhs(ib_ctx *c, const double *u, const double *F, double *r_out) {
  if (c && c->slab_P) return fail(IB_ESTATE, "debug entry points need a whole-lattice context");
  if (!c || !u || !F || !r_out) return fail(IB_EINVAL, "NULL argument");
  Tmp t; double *ud, *Fd, *r;
  const size_t V = (size_t)c->g.V;
  CK(t.get(&ud, 3 * V)); CK(t.get(&Fd, 3 * V)); CK(t.get(&r, 3 * V));
  CK(copy_sync(ud, u, 3 * V * sizeof(double), c->stream));
  CK(copy_sync(Fd, F, 3 * V * sizeof(double), c->stream));
  CK(xfwd(c, 1, ud, Fd, nullptr, r, c->stream));
  CK(copy_sync(r_out, r, 3 * V * sizeof(double), c->stream));
  return IB_OK;
}

int ib_debug_fluid(ib_ctx *c, const double *u, const double *F, double *u_out, double *p_out) {
  if (c && c->slab_P) return fail(IB_ESTATE, "debug entry points need a whole-lattice context");
  if (!c || !u || !F || !u_out) return fail(IB_EINVAL, "NULL argument");
  Tmp t; double *ud, *Fd, *pd = nullptr; double2 *ps = nullptr, *ps1 = nullptr;
  const FluidGeom &g = c->g;
  const size_t V = (size_t)g.V;
  cudaStream_t s = c->stream;
  CK(t.get(&ud, 3 * V)); CK(t.get(&Fd, 3 * V));
  if (p_out) {
    CK(t.get(&ps, pspec_elems(c))); CK(t.get(&ps1, spec1_elems(c)));
    CK(t.get(&pd, V));
  }
  CK(copy_sync(ud, u, 3 * V * sizeof(double), s));
  CK(copy_sync(Fd, F, 3 * V * sizeof(double), s));
  CK(xfwd(c, 0, ud, Fd, nullptr, nullptr, s));
  CK(yfwd(c, s));
  CK(zsolve(c, ps, s));
  CK(yinv(c, s));
  CK(xinv(c, ud, nullptr, 0, nullptr, s));
  if (p_out) {
    CK(pressure_to_real(c, ps, ps1, pd, s));
    CK(copy_sync(p_out, pd, V * sizeof(double), s));
  }
  CK(copy_sync(u_out, ud, 3 * V * sizeof(double), s));
  return IB_OK;
}

namespace {
__global__ void k_scale(double *a, size_t n, double f) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    a[i] *= f;
}
}  // namespace

// S3c alone: u^, p^ from r^ (half spectra [3][N3][N2][N1/2+1] / [N3][N2][N1/2+1], complex
// interleaved).  Runs the product z kernel (forward z, per-mode solve, inverse z) between an
// inverse and a forward z transform, so the solve sees r^ (times N3); the scale factors of the
// unnormalised transforms and of the solve's folded 1/V are undone.  Needs the TMA z pass
// (N3 in [64, 512]).
int ib_debug_project(ib_ctx *c, const double *rhat, double *uhat, double *phat) {
  if (c && c->slab_P) return fail(IB_ESTATE, "debug entry points need a whole-lattice context");
  if (!c || !rhat || !uhat) return fail(IB_EINVAL, "NULL argument");
  if (!c->maps.z_ok) return fail(IB_ESTATE, "ib_debug_project needs N3 in [64, 512]");
  const FluidGeom &g = c->g;
  cudaStream_t s = c->stream;
  const size_t H = (size_t)(g.M + 1), row = H * 2 * sizeof(double);
  Tmp t; double2 *ps;
  CK(t.get(&ps, pspec_elems(c)));
  for (int comp = 0; comp < 3; ++comp)      // [comp][kz][ky][kx] -> S2 [comp][ky][kz][kx]
    for (int ky = 0; ky < g.N2; ++ky)
      CK(cudaMemcpy2DAsync(c->spec2 + ((size_t)comp * g.N2 + ky) * g.N3 * g.P, (size_t)g.P * sizeof(double2),
                           rhat + (((size_t)comp * g.N3) * g.N2 + ky) * H * 2, (size_t)g.N2 * row,
                           row, (size_t)g.N3, cudaMemcpyDefault, s));
  const Sym sy = sym_of(c);
  CK(launch_colfft(g, 4, c->maps, nullptr, c->tw[2], sy, s));    // inverse z
  CK(launch_colfft(g, 0, c->maps, ps, c->tw[2], sy, s));         // z, solve, inverse z
  CK(launch_colfft(g, 3, c->maps, nullptr, c->tw[2], sy, s));    // forward z
  // unnormalised z transforms around the solve (which folds in 1/V): u^ comes out scaled by
  // N3^2 / V, p^ (written at solve time, between the z transforms) by N3 / V
  const double V = (double)g.V, N3 = (double)g.N3;
  k_scale<<<592, 256, 0, s>>>(reinterpret_cast<double *>(c->spec2), 3 * spec1_elems(c) * 2, V / (N3 * N3));
  k_scale<<<592, 256, 0, s>>>(reinterpret_cast<double *>(ps), spec1_elems(c) * 2, V / N3);
  c->launches += 5;
  for (int comp = 0; comp < 3; ++comp)      // S2 -> [comp][kz][ky][kx]
    for (int ky = 0; ky < g.N2; ++ky)
      CK(cudaMemcpy2DAsync(uhat + (((size_t)comp * g.N3) * g.N2 + ky) * H * 2, (size_t)g.N2 * row,
                           c->spec2 + ((size_t)comp * g.N2 + ky) * g.N3 * g.P, (size_t)g.P * sizeof(double2),
                           row, (size_t)g.N3, cudaMemcpyDefault, s));
  if (phat)
    for (int ky = 0; ky < g.N2; ++ky)
      CK(cudaMemcpy2DAsync(phat + (size_t)ky * H * 2, (size_t)g.N2 * row,
                           ps + (size_t)ky * g.N3 * g.P, (size_t)g.P * sizeof(double2),
                           row, (size_t)g.N3, cudaMemcpyDefault, s));
  CK(cudaStreamSynchronize(s));
  return IB_OK;
}

// S3d alone: unnormalised inverse 3-D DFT of a half spectrum in [N3][N2][N1/2+1] (complex
// interleaved) -> real out [V], through the product inverse passes (z, y, then the x C2R),
// i.e. sum_k X_k e^{+2 pi i sum k_a j_a / N_a} over the full Hermitian spectrum.  The TMA
// column passes transform 3 component slots; slot 0 carries the data.
int ib_debug_ifft(ib_ctx *c, const double *in, double *out) {
  if (c && c->slab_P) return fail(IB_ESTATE, "debug entry points need a whole-lattice context");
  if (!c || !in || !out) return fail(IB_EINVAL, "NULL argument");
  const FluidGeom &g = c->g;
  cudaStream_t s = c->stream;
  const size_t H = (size_t)(g.M + 1), row = H * 2 * sizeof(double);
  CK(cudaMemsetAsync(c->spec2, 0, 3 * spec1_elems(c) * sizeof(double2), s));
  for (int ky = 0; ky < g.N2; ++ky)          // [kz][ky][kx] -> S2 slot 0 [ky][kz][kx]
    CK(cudaMemcpy2DAsync(c->spec2 + (size_t)ky * g.N3 * g.P, (size_t)g.P * sizeof(double2),
                         in + (size_t)ky * H * 2, (size_t)g.N2 * row, row, (size_t)g.N3,
                         cudaMemcpyDefault, s));
  Tmp t; double *o;
  CK(t.get(&o, 3 * (size_t)g.V));
  if (c->maps.z_ok) {
    CK(launch_colfft(g, 4, c->maps, nullptr, c->tw[2], sym_of(c), s));
  } else {                                   // inverse z through the pressure path's pass
    return fail(IB_ESTATE, "ib_debug_ifft needs N3 in [64, 512]");
  }
  CK(yinv(c, s));
  CK(xinv(c, o, nullptr, 0, nullptr, s));
  c->launches += 3;
  CK(copy_sync(out, o, (size_t)g.V * sizeof(double), s));
  return IB_OK;
}

int ib_debug_fft(ib_ctx *c, const double *in, double *out) {
  if (c && c->slab_P) return fail(IB_ESTATE, "debug entry points need a whole-lattice context");
  if (!c || !in || !out) return fail(IB_EINVAL, "NULL argument");
  Tmp t; double *ind;
  const FluidGeom &g = c->g;
  const size_t V = (size_t)g.V;
  cudaStream_t s = c->stream;
  CK(t.get(&ind, V));
  CK(copy_sync(ind, in, V * sizeof(double), s));
  CK(xfwd(c, 2, ind, nullptr, nullptr, nullptr, s));
  // (TMA passes transform all 3 component slots; only slot 0 is read)
  if (c->maps.y_ok) CK(launch_colfft(g, 1, c->maps, nullptr, c->tw[1], sym_of(c), s));
  else CK(launch_ypass(g, -1, c->spec, 1, c->spec2, 2, 1, c->tw[1], s));
  if (c->maps.z_ok) CK(launch_colfft(g, 3, c->maps, nullptr, c->tw[2], sym_of(c), s));
  else CK(launch_zpass(g, 1, c->spec2, nullptr, c->tw[2], sym_of(c), s));
  // S2 [ky][kz][kx] -> out [kz][ky][kx]
  for (int ky = 0; ky < g.N2; ++ky)
    CK(cudaMemcpy2DAsync(out + (size_t)ky * (g.M + 1) * 2, (size_t)g.N2 * (g.M + 1) * 2 * sizeof(double),
                         c->spec2 + (size_t)ky * g.N3 * g.P, (size_t)g.P * sizeof(double2),
                         (size_t)(g.M + 1) * sizeof(double2), (size_t)g.N3, cudaMemcpyDefault, s));
  CK(cudaStreamSynchronize(s));
  return IB_OK;
}

}  // extern "C"
