// mma_rate.cu — dev microbenchmark: tcgen05.mma (kind::f16, bf16 -> fp32) issue rate per SM
// for the shapes / operand sources the attention kernels use. One CTA per SM, one thread
// issues NI MMAs (K = 16 each) back to back into TMEM, commit, wait; clock64 delta / NI.
// Operand contents are whatever smem holds (throughput only).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/mma_rate bench_tools/mma_rate.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../paper_2603_18567_b200/csrc/ptx_sm100.cuh"
using namespace tttk;

// MODE: 0 SS (A K-major, B K-major), 1 SS (A MN-major, B MN-major), 2 TS (A TMEM, B MN-major)
// NACC: number of distinct TMEM accumulators the MMAs rotate over (1 = one dependent chain)
template <int MODE, int M, int N, int NACC>
__global__ void __launch_bounds__(128, 1) rate_kernel(int NI, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc(&tb, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tb;
  if (warp == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    const uint64_t da = MODE == 1 ? sdesc_sw128(a, 16384, 1024) : sdesc_sw128(a, 16, 1024);
    const uint64_t db = MODE == 0 ? sdesc_sw128(b, 16, 1024) : sdesc_sw128(b, 16384, 1024);
    constexpr uint32_t id = idesc_bf16_f32(M, N, MODE == 1, MODE != 0);
    constexpr uint32_t dstride = NACC == 1 ? 0 : (MODE == 2 ? 64 : 128);
    for (int rep = 0; rep < 2; ++rep) {
      __syncwarp();
      const long long t0 = clock64();
      for (int i = 0; i < NI; i += 8) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint32_t d = tbase + (MODE == 2 ? 256 : 0) + dstride * (ks % NACC);
          if (MODE == 2)
            umma_ts_e(d, tbase + 8 * ks, sdesc_add(db, ks * 2048), id, 1);
          else if (MODE == 0)
            umma_ss_e(d, sdesc_add(da, (ks & 3) * 32), sdesc_add(db, (ks & 3) * 32), id, 1);
          else
            umma_ss_e(d, sdesc_add(da, ks * 2048), sdesc_add(db, ks * 2048), id, 1);
        }
      }
      umma_commit_e(&bar);
      mbar_wait(&bar, rep & 1);
      const long long t1 = clock64();
      if (rep == 1 && threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

template <int MODE, int M, int N, int NACC>
void run(const char* name, unsigned long long* d, int grid) {
  const int NI = 4096;
  cudaFuncSetAttribute(rate_kernel<MODE, M, N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  rate_kernel<MODE, M, N, NACC><<<grid, 128, 200 * 1024>>>(NI, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s error %s\n", name, cudaGetErrorString(e)); exit(1); }
  unsigned long long h[148];
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < grid; ++i) s += h[i];
  const double cyc = s / grid / NI;
  const double floor_ = (M < 128 ? 128 : M) * N / 256.0;
  printf("%-26s nacc=%d grid=%3d  %6.1f cyc/mma (floor %5.1f)  %5.0f flop/clk/SM\n", name, NACC, grid, cyc, floor_,
         2.0 * M * N * 16 / cyc);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  for (int grid : {1, 148}) {
    run<0, 128, 64, 1>("SS K-major   M128 N64", d, grid);
    run<0, 128, 64, 4>("SS K-major   M128 N64", d, grid);
    run<0, 128, 128, 1>("SS K-major   M128 N128", d, grid);
    run<0, 128, 128, 4>("SS K-major   M128 N128", d, grid);
    run<0, 128, 256, 1>("SS K-major   M128 N256", d, grid);
    run<1, 128, 64, 1>("SS MN-major  M128 N64", d, grid);
    run<1, 128, 128, 1>("SS MN-major  M128 N128", d, grid);
    run<2, 128, 64, 1>("TS B MN      M128 N64", d, grid);
    run<2, 128, 64, 4>("TS B MN      M128 N64", d, grid);
    run<2, 128, 128, 1>("TS B MN      M128 N128", d, grid);
    run<2, 128, 128, 2>("TS B MN      M128 N128", d, grid);
    run<2, 128, 256, 1>("TS B MN      M128 N256", d, grid);
    run<0, 64, 128, 1>("SS K-major   M64  N128", d, grid);
  }
  return 0;
}
