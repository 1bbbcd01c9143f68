// slab.cu — the IB step decomposed into P slabs of the lattice along z (SURVEY.md §8(e),
// §8(f) row 4).  The paper partitions the fluid and material grids over its
// processors (PAPER.md 801-807) and names the 2x refined model that needs it (1238-1245).
//
// Rank r of P owns the planes z in [r L, (r + 1) L), L = N3 / P.  One step is five phases on
// the context stream with a caller-driven exchange between them (NCCL collectives across
// processes, or device copies between contexts of one process):
//   0  force + spread onto the owned planes, x forward (rhs + R2C), y forward -> S2
//        [caller: per component, all-to-all S2 [dst][Ky][L] -> Z [src][Ky][L]]
//   1  z forward FFT + per-mode solve + z inverse on the received blocks Z (5-D TMA map)
//        [caller: per component, all-to-all Z -> S2]
//   2  y inverse, x inverse (C2R) -> owned planes of u; the edge planes (last, first,
//      second owned) are copied to edge_send
//        [caller: all-gather edge_send -> edge_recv [P]]
//   3  ghost planes of u from the neighbours' edges (1 below, 2 above: the upwind rhs needs
//      z +- 1, the interpolation window floor - 1 .. floor + 2); interpolation + update of
//      the owned points (base plane in the slab), packed as (x, y, z, index) records
//        [caller: all-gather count_send -> count_recv, pack_send -> pack_recv]
//   4  every rank's records scattered into this rank's replica of X; step counter + 1
// With ib_slab_set_peers the two transposes are fused into the kernels: phase 0's y-forward
// pass stores each tile's Ky-row block bound for rank d straight into rank d's Z, phase 1's
// z solve each L-row block of source rank d straight into rank d's S2 (TMA stores through
// per-peer maps), and the caller only orders the ranks after phases 0 and 1.
// Positions are replicated on every rank; each rank computes the forces of the points whose
// support meets its planes and spreads only onto its own planes, so the spread needs no
// halo reduction.
#include <climits>
#include <cstring>
#include <string>

#include "api.cuh"

using namespace ibk;

namespace {

__global__ void k_scatter_pack(const double4 *__restrict__ recv, const unsigned long long *counts,
                               int P, int64_t cap, double *X, int64_t np) {
  const int src = blockIdx.y;
  if (src >= P) return;
  const unsigned long long cnt = counts[src];
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < (int64_t)cnt;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double4 r = recv[(size_t)src * cap + k];
    const int64_t i = (int64_t)r.w;
    if (i >= 0 && i < np) {
      X[3 * i + 0] = r.x; X[3 * i + 1] = r.y; X[3 * i + 2] = r.z;
    }
  }
}

bool slab_dims_ok(int32_t N1, int32_t N2, int32_t N3, int32_t P, int32_t rank, std::string &why) {
  auto p2 = [](int n) { return n > 0 && !(n & (n - 1)); };
  if (!(N1 >= 64 && N1 <= 512 && N2 >= 64 && N2 <= 512 && N3 >= 64 && N3 <= 512) ||
      !p2(N1) || !p2(N2) || !p2(N3)) {
    why = "slab lattices need N1, N2, N3 powers of two in [64, 512] (TMA passes)";
    return false;
  }
  if (P < 1 || !p2(P) || rank < 0 || rank >= P) { why = "P must be a power of two, 0 <= rank < P"; return false; }
  if (N3 % P || N3 / P < 8) { why = "L = N3 / P must be >= 8"; return false; }
  if (N2 % P) { why = "N2 must be a multiple of P (the z pass splits ky)"; return false; }
  return true;
}

}  // namespace

extern "C" {

ib_ctx *ib_slab_create(int32_t N1, int32_t N2, int32_t N3, double h, double rho, double mu,
                       double dt, int32_t P, int32_t rank) {
  std::string why;
  if (!slab_dims_ok(N1, N2, N3, P, rank, why)) {
    fail(IB_EINVAL, why);
    return nullptr;
  }
  const int L = N3 / P, Ky = N2 / P;
  ib_ctx *c = ib_create3(N1, N2, L, h, rho, mu, dt);   // local planes: x, y passes, spread
  if (!c) return nullptr;
  auto bad = [&](cudaError_t e, const char *what) {
    fail(e == cudaErrorMemoryAllocation ? IB_ENOMEM : IB_ECUDA,
         std::string("ib_slab_create: ") + what + ": " + cudaGetErrorString(e));
    ib_destroy(c);
    return (ib_ctx *)nullptr;
  };
  FluidGeom &g = c->g;
  g.N3g = N3;
  g.Vg = (int64_t)N1 * N2 * N3;
  g.z0 = rank * L;
  g.uz0 = 1;
  g.uN3 = L + 3;
  g.L = L;
  g.slab = 1;
  c->gz = g;                                 // z pass: Ky local ky rows, whole z pencils
  c->gz.N2 = Ky;
  c->gz.N3 = N3;
  c->gz.V = (int64_t)N1 * Ky * N3;
  c->gz.ky0 = rank * Ky;
  c->gz.z0 = 0;
  c->gz.uz0 = 0;
  c->gz.uN3 = N3;
  c->slab_P = P;
  c->slab_rank = rank;
  cudaError_t e;
  // velocity with its ghost planes: [3][L + 3][N2][N1], local plane z at 1 + z
  dfree(c->u);
  c->u = nullptr;
  const size_t Vu = (size_t)N1 * N2 * (L + 3);
  if ((e = dalloc(&c->u, 3 * Vu)) != cudaSuccess) return bad(e, "u");
  if ((e = cudaMemsetAsync(c->u, 0, 3 * Vu * sizeof(double), c->stream)) != cudaSuccess) return bad(e, "memset");
  dfree(c->spec2);                           // S2 is a caller buffer (ib_slab_set_buffers)
  c->spec2 = nullptr;
  c->maps.y_ok = c->maps.z_ok = false;
  // z axis tables of the whole pencil length N3
  dfree(c->tw[2]); dfree(c->sym_s[2]); dfree(c->sym_l[2]);
  c->tw[2] = nullptr; c->sym_s[2] = c->sym_l[2] = nullptr;
  if ((e = dalloc(&c->tw[2], (size_t)N3)) != cudaSuccess) return bad(e, "tables");
  if ((e = dalloc(&c->sym_s[2], (size_t)N3)) != cudaSuccess) return bad(e, "tables");
  if ((e = dalloc(&c->sym_l[2], (size_t)N3)) != cudaSuccess) return bad(e, "tables");
  if ((e = init_axis_table(c->tw[2], N3, c->sym_s[2], c->sym_l[2], h, c->stream)) != cudaSuccess)
    return bad(e, "tables");
  c->launches++;
  if ((e = fluid_setup_attributes(N3)) != cudaSuccess) return bad(e, "attributes");
  // x forward reads the ghosted u
  c->umaps.ok = false;
  xfwd_encode_u(c->g, c->u, &c->umaps);
  // device step counter and non-finite flag live across phase calls
  *c->flag_h = LLONG_MAX;
  if ((e = cudaMemcpyAsync(c->flag, c->flag_h, sizeof(long long), cudaMemcpyHostToDevice, c->stream)) != cudaSuccess)
    return bad(e, "flag");
  if ((e = cudaMemsetAsync(c->dev_n, 0, sizeof(long long), c->stream)) != cudaSuccess) return bad(e, "counter");
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return bad(e, "sync");
  return c;
}

int ib_slab_info(ib_ctx *c, int32_t *info, int32_t cap) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  if (!c->slab_P) return fail(IB_ESTATE, "not a slab context");
  const int32_t v[8] = {c->slab_P, c->slab_rank, c->g.L, c->gz.N2, c->g.N1, c->g.N2g, c->g.N3g,
                        c->g.P};
  for (int k = 0; k < cap && k < 8; ++k) info[k] = v[k];
  return IB_OK;
}

int ib_slab_set_buffers(ib_ctx *c, void *s2, void *z, double *edge_send, double *edge_recv,
                        void *pack_send, void *pack_recv, uint64_t *count_send,
                        uint64_t *count_recv, int64_t pack_cap) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  if (!c->slab_P) return fail(IB_ESTATE, "not a slab context");
  if (!s2 || !z || !edge_send || !edge_recv || !pack_send || !pack_recv || !count_send ||
      !count_recv)
    return fail(IB_EINVAL, "NULL buffer");
  if (pack_cap < c->np) return fail(IB_EINVAL, "pack_cap must be >= np");
  CK(cudaStreamSynchronize(c->stream));
  c->s2_ext = static_cast<double2 *>(s2);
  c->z_ext = static_cast<double2 *>(z);
  c->edge_send = edge_send;
  c->edge_recv = edge_recv;
  c->pack_send = static_cast<double4 *>(pack_send);
  c->pack_recv = static_cast<double4 *>(pack_recv);
  c->count_send = reinterpret_cast<unsigned long long *>(count_send);
  c->count_recv = reinterpret_cast<unsigned long long *>(count_recv);
  c->pack_cap = pack_cap;
  TmaMaps m;
  CK(colfft_make_maps(c->g, c->spec, c->s2_ext, &m));       // y passes: S1 <-> S2 (local planes)
  if (!m.y_ok) return fail(IB_EINVAL, "y passes need N2 in [64, 512]");
  m.z_ok = false;
  c->maps = m;
  TmaMaps zm;
  if (!colfft_encode_slabz(c->gz, c->z_ext, c->slab_P, &zm.s2_2d))
    return fail(IB_EINVAL, "z pass map of the received blocks");
  zm.z_ok = true;
  c->zmaps = zm;
  return IB_OK;
}

int ib_slab_set_peers(ib_ctx *c, int32_t P, void *const *s2_peers, void *const *z_peers) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  if (!c->slab_P) return fail(IB_ESTATE, "not a slab context");
  if (!c->z_ext) return fail(IB_ESTATE, "ib_slab_set_buffers first");
  CK(cudaStreamSynchronize(c->stream));
  if (P == 0) {
    c->maps.peers.P = 0;
    c->zmaps.peers.P = 0;
    return IB_OK;
  }
  if (P != c->slab_P) return fail(IB_EINVAL, "P must equal the slab count");
  if (P > MAX_PEERS) return fail(IB_EINVAL, "at most " + std::to_string(MAX_PEERS) + " peers");
  if (!s2_peers || !z_peers) return fail(IB_EINVAL, "NULL peer array");
  for (int d = 0; d < P; ++d)
    if (!s2_peers[d] || !z_peers[d]) return fail(IB_EINVAL, "NULL peer buffer");
  const int L = c->g.L, Ky = c->gz.N2, r = c->slab_rank;
  const int cy = 8, cz = c->gz.N3 >= 128 ? 4 : 8;   // the y / z tiles' columns (fluid_tma.cu)
  PeerMaps y{}, z{};
  for (int d = 0; d < P; ++d) {
    if (!colfft_encode_peer(c->gz, static_cast<double2 *>(z_peers[d]), P, r, cy, 1, Ky, &y.m[d]) ||
        !colfft_encode_peer(c->gz, static_cast<double2 *>(s2_peers[d]), P, r, cz, L, 1, &z.m[d]))
      return fail(IB_EINVAL, "peer TMA maps");
  }
  y.P = z.P = P;
  y.rows = Ky;
  z.rows = L;
  c->maps.peers = y;
  c->zmaps.peers = z;
  return IB_OK;
}

int ib_slab_phase(ib_ctx *c, int32_t phase) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  if (!c->slab_P) return fail(IB_ESTATE, "not a slab context");
  if (!c->z_ext) return fail(IB_ESTATE, "ib_slab_set_buffers first");
  if (c->np > c->pack_cap) return fail(IB_ESTATE, "structure larger than pack_cap");
  if (phase != c->slab_next)                 // the exchanges between phases assume the order
    return fail(IB_ESTATE, "slab phase " + std::to_string(phase) + " called, expected " +
                               std::to_string(c->slab_next));
  c->slab_next = (c->slab_next + 1) % 5;
  const FluidGeom &g = c->g;
  cudaStream_t s = c->stream;
  const size_t plane = (size_t)g.N1 * g.N2;
  const size_t Vu = plane * g.uN3;
  const int L = g.L, P = c->slab_P, r = c->slab_rank;
  switch (phase) {
    case 0: {
      CK(ensure_binned(c, s));
      CK(launch_force_spread(struct_dev(c), g, nullptr, c->dev_n, 0, c->F, c->rowflag, s));
      CK(xfwd(c, 0, c->u, c->F, c->rowflag, nullptr, s));
      CK(yfwd(c, s));
      c->launches += 2 + (c->np > 0 ? 1 : 0);   // the drive runs inside the spread
      return IB_OK;
    }
    case 1:
      CK(launch_colfft(c->gz, 0, c->zmaps, nullptr, c->tw[2], sym_of(c), s));
      c->launches += 1;
      return IB_OK;
    case 2: {
      CK(yinv(c, s));
      CK(xinv(c, c->u, c->dev_n, 0, c->flag, s));
      c->launches += 2;
      const int pl[3] = {L - 1, 0, 1};         // last, first, second owned plane
      for (int k = 0; k < 3; ++k)
        for (int comp = 0; comp < 3; ++comp)
          CK(cudaMemcpyAsync(c->edge_send + (k * 3 + comp) * plane,
                             c->u + comp * Vu + (size_t)(g.uz0 + pl[k]) * plane,
                             plane * sizeof(double), cudaMemcpyDeviceToDevice, s));
      return IB_OK;
    }
    case 3: {
      const int prev = (r - 1 + P) % P, next = (r + 1) % P;
      const size_t edge = 9 * plane;               // one rank's edge block
      // ghost plane uz0 - 1 = z0 - 1 (prev's last), uz0 + L = z0 + L (next's first),
      // uz0 + L + 1 = z0 + L + 1 (next's second)
      const int dst[3] = {g.uz0 - 1, g.uz0 + L, g.uz0 + L + 1};
      const int src_rank[3] = {prev, next, next};
      for (int k = 0; k < 3; ++k)
        for (int comp = 0; comp < 3; ++comp)
          CK(cudaMemcpyAsync(c->u + comp * Vu + (size_t)dst[k] * plane,
                             c->edge_recv + src_rank[k] * edge + (k * 3 + comp) * plane,
                             plane * sizeof(double), cudaMemcpyDeviceToDevice, s));
      CK(cudaMemsetAsync(c->count_send, 0, sizeof(unsigned long long), s));
      CK(launch_interp(g, c->u, c->X, c->np, nullptr, c->flag, c->dev_n, 0,
                       c->since_bin >= 0 ? c->perm : nullptr, c->fixed, s, c->pack_send,
                       c->count_send, c->Xs));
      if (c->np > 0) c->launches += 1;
      return IB_OK;
    }
    case 4: {
      if (c->np > 0) {
        const int64_t per = c->np / P + 1;
        dim3 grid((unsigned)((per + 255) / 256 < 1184 ? (per + 255) / 256 : 1184), (unsigned)P);
        k_scatter_pack<<<grid, 256, 0, s>>>(c->pack_recv, c->count_recv, P, c->pack_cap, c->X,
                                            c->np);
        CK(cudaGetLastError());
        c->launches += 1;
        if (c->since_bin >= 0) {                 // the binned copy follows the other ranks' points
          CK(launch_gather_xs(c->X, c->perm, c->np, c->Xs, s));
          c->launches += 1;
        }
      }
      CK(launch_step_inc(c->dev_n, s));
      c->launches += 1;
      c->n += 1;
      c->since_bin++;
      return IB_OK;
    }
    default:
      return fail(IB_EINVAL, "phase must be 0..4");
  }
}

int ib_slab_sync(ib_ctx *c) {
  if (!c) return fail(IB_EINVAL, "ctx is NULL");
  if (!c->slab_P) return fail(IB_ESTATE, "not a slab context");
  CK(cudaMemcpyAsync(c->flag_h, c->flag, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const long long bad = *c->flag_h;
  if (bad != LLONG_MAX) {
    *c->flag_h = LLONG_MAX;
    CK(cudaMemcpyAsync(c->flag, c->flag_h, sizeof(long long), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return fail(IB_ENONFINITE, "non-finite u or X first at step " + std::to_string(bad));
  }
  return IB_OK;
}

}  // extern "C"
