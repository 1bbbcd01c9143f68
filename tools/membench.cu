// membench.cu — DRAM efficiency of the strided-pencil access patterns used by the FFT passes.
// A CTA copies a tile of W consecutive 16-byte elements x H rows (row pitch PITCH bytes)
// from src to dst; lanes are W-fastest, so one warp instruction touches 32/W rows of W*16
// bytes.  Reports GB/s (read + write) for several W and pitches.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/membench tools/membench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int W, int H, int ILP>
__global__ void k_tile(const double2 *__restrict__ src, double2 *__restrict__ dst,
                       size_t pitch_el, int tiles_x) {
  const int col = threadIdx.x % W, r0 = threadIdx.x / W;
  constexpr int RPI = 256 / W;    // rows covered by the CTA per iteration (256 threads)
  const size_t tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
  const size_t base = ty * H * pitch_el + tx * W + col;
  double2 v[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) v[i] = src[base + (size_t)(r0 + i * RPI) * pitch_el];
#pragma unroll
  for (int i = 0; i < ILP; ++i) dst[base + (size_t)(r0 + i * RPI) * pitch_el] = v[i];
}

template <int W>
void run(size_t pitch_bytes, double2 *a, double2 *b, size_t total_bytes) {
  constexpr int ILP = 16, H = (256 / W) * ILP;
  const size_t pitch_el = pitch_bytes / 16;
  const int tiles_x = (int)(pitch_el / W);
  const size_t rows = total_bytes / pitch_bytes;
  const int tiles_y = (int)(rows / H);
  const int grid = tiles_x * tiles_y;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k_tile<W, H, ILP><<<grid, 256>>>(a, b, pitch_el, tiles_x);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int w = 0; w < reps; ++w) k_tile<W, H, ILP><<<grid, 256>>>(a, b, pitch_el, tiles_x);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = 2.0 * (double)grid * 256 * ILP * 16;
  printf("W=%2d seg=%4dB pitch=%8zuB  %7.1f GB/s\n", W, W * 16, pitch_bytes,
         bytes * reps / (ms * 1e-3) / 1e9);
}

int main() {
  const size_t total = (size_t)1 << 30;   // 1 GiB each way
  double2 *a, *b;
  cudaMalloc(&a, total + (64 << 20));
  cudaMalloc(&b, total + (64 << 20));
  cudaMemset(a, 0, total); cudaMemset(b, 0, total);
  const size_t pitches[] = {2048, 2080, 532480, 4096 * 129};
  for (size_t p : pitches) {
    run<2>(p, a, b, total); run<4>(p, a, b, total); run<8>(p, a, b, total);
    run<16>(p, a, b, total); run<32>(p, a, b, total);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
