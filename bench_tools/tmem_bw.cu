// tmem_bw.cu — dev microbenchmark: tcgen05.ld / tcgen05.st throughput per SM (bytes per clock)
// for the load shapes the attention kernels use (32x32b.x32 / .x64-as-2, one wait per batch).
// One CTA per SM, W warps; warp w reads TMEM lanes of quadrant w % 4 (the hardware rule), a
// different column window per warp. Reports clk per load and B/clk/SM for the whole CTA.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/tmem_bw bench_tools/tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../paper_2603_18567_b200/csrc/ptx_sm100.cuh"
using namespace tttk;

// MODE 0: ld x32 + wait per load; 1: two x32 loads then one wait (tmem_ld64w); 2: four x32 + wait;
// MODE 3: st x32 + wait::st per store
template <int MODE>
__global__ void __launch_bounds__(512, 1) bw_kernel(int NI, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) { tmem_alloc(&tb, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tb;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t col0 = (uint32_t)((warp >> 2) * 128);  // 4 column windows of 128
  uint32_t acc = 0;
  long long t0 = 0, t1 = 0;
  for (int rep = 0; rep < 2; ++rep) {
    __syncthreads();
    t0 = clock64();
    for (int i = 0; i < NI; ++i) {
      const uint32_t a = tbase + lane_off + col0 + (uint32_t)((i & 1) * 64);
      if (MODE == 0) {
        uint32_t r[32];
        tmem_ld32(a, r);
#pragma unroll
        for (int k = 0; k < 32; ++k) acc ^= r[k];
      } else if (MODE == 1) {
        uint32_t r[64];
        tmem_ld64w(a, r);
#pragma unroll
        for (int k = 0; k < 64; ++k) acc ^= r[k];
      } else if (MODE == 2) {
        uint32_t r[64], s[64];
        tmem_ld64w(a, r);
        tmem_ld64w(a ^ 64, s);
#pragma unroll
        for (int k = 0; k < 64; ++k) acc ^= r[k] ^ s[k];
      } else {
        uint32_t r[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) r[k] = acc + k + i;
        tmem_st32(a, r);
        tmem_st_wait();
        acc += 1;
      }
    }
    __syncthreads();
    t1 = clock64();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

template <int MODE>
void run(const char* name, int warps, int grid, unsigned long long* d, uint32_t* sink) {
  const int NI = 2048;
  bw_kernel<MODE><<<grid, warps * 32>>>(NI, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s error %s\n", name, cudaGetErrorString(e)); exit(1); }
  unsigned long long h[148];
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < grid; ++i) s += h[i];
  const double cyc = s / grid;
  const double bytes_per_iter = (MODE == 0 || MODE == 3 ? 32 : MODE == 1 ? 64 : 128) * 4.0 * 32;  // per warp
  const double bpc = bytes_per_iter * NI * warps / cyc;
  printf("%-28s warps=%2d grid=%3d  %8.1f clk per iter per warp  %7.1f B/clk/SM\n", name, warps, grid, cyc / NI, bpc);
}

int main() {
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 512 * 4);
  for (int grid : {1, 148})
    for (int w : {4, 8, 16}) {
      run<0>("ld 32x32b.x32 + wait", w, grid, d, sink);
      run<1>("ld 2 x x32 + wait", w, grid, d, sink);
      run<2>("ld 4 x x32 + 2 waits", w, grid, d, sink);
      run<3>("st 32x32b.x32 + wait", w, grid, d, sink);
    }
  return 0;
}
