// kbench.cu — dev micro-benchmark of the fluid-pass launchers in libib_b200.so (N = 256).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build_variants/kbench \
//      tools/kbench.cu -Lpaper_math_0301321_b200 -lib_b200 -Xlinker -rpath,$PWD/paper_math_0301321_b200
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_math_0301321_b200/csrc/ib_internal.cuh"

using namespace ibk;

template <class F>
float timeit(F f, int reps = 20) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return 1e3f * ms / reps;
}

int main(int argc, char **argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 256;
  ib_ctx *c = ib_create(N, 1.0 / N, 1.0, 1e-3, 1e-4);
  if (!c) { printf("create failed: %s\n", ib_last_error()); return 1; }
  const FluidGeom &g = c->g;
  cudaStream_t s = 0;
  const double C = (double)N * N * (N / 2 + 1), V = (double)N * N * N;
  auto rep = [&](const char *n, float us, double bytes) {
    printf("%-28s %8.1f us  %7.0f GB/s\n", n, us, bytes / (us * 1e-6) / 1e9);
  };
  rep("xfwd (rhs+r2c)", timeit([&] { launch_xfwd(g, 0, c->u, c->F, c->rowflag, nullptr, nullptr, c->spec, c->twN, c->twM, s); }), 24 * V + 48 * C);
  rep("xfwd mode2 (r2c only,1c)", timeit([&] { launch_xfwd(g, 2, nullptr, nullptr, nullptr, c->u, nullptr, c->spec, c->twN, c->twM, s); }), 8 * V + 16 * C);
  rep("y fwd S1->S2", timeit([&] { launch_ypass(g, -1, c->spec, 1, c->spec2, 2, 3, c->twN, s); }), 96 * C);
  rep("y inv S2->S1", timeit([&] { launch_ypass(g, +1, c->spec2, 2, c->spec, 1, 3, c->twN, s); }), 96 * C);
  rep("y S1->S1", timeit([&] { launch_ypass(g, -1, c->spec, 1, c->spec, 1, 3, c->twN, s); }), 96 * C);
  rep("y S2->S2", timeit([&] { launch_ypass(g, -1, c->spec2, 2, c->spec2, 2, 3, c->twN, s); }), 96 * C);
  rep("z fwd only (mode 1)", timeit([&] { launch_zpass(g, 1, c->spec2, nullptr, c->twN, c->sym_s, c->sym_l, s); }), 96 * C);
  rep("z fwd+solve+inv", timeit([&] { launch_zpass(g, 0, c->spec2, nullptr, c->twN, c->sym_s, c->sym_l, s); }), 96 * C);
  rep("xinv (c2r)", timeit([&] { launch_xinv(g, c->spec, c->u, 3, c->twN, c->twM, nullptr, nullptr, 0, s); }), 48 * C + 24 * V);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  ib_destroy(c);
  return 0;
}
