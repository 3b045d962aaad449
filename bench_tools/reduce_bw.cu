// reduce_bw.cu — dev microbenchmark: TMA bulk reduce-add (fp32 add, 32 x 32 SW128 boxes of 4 KB,
// the bwd kernel's dQ path) and plain TMA bulk store of the same boxes, per-SM and chip-wide
// throughput vs the number of CTAs. Each CTA keeps up to 8 boxes in flight (wait_group.read).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/reduce_bw bench_tools/reduce_bw.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../paper_2603_18567_b200/csrc/ptx_sm100.cuh"
using namespace tttk;

__global__ void __launch_bounds__(32, 1) red_kernel(const __grid_constant__ CUtensorMap m, int nbox_total, int iters,
                                                    int store, int brows, int hot, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (threadIdx.x != 0) return;
  const int bbytes = brows * 128;
  for (int i = 0; i < 8 * bbytes / 4; ++i) reinterpret_cast<float*>(smem)[i] = 1.f;
  fence_async_smem();
  const long long t0 = clock64();
  uint32_t rng = 777u + blockIdx.x * 7919u;
  for (int it = 0; it < iters; ++it) {
    if (it >= 8) bulk_wait_group_read<7>();
    rng = rng * 1664525u + 1013904223u;
    const int nb = hot ? 2048 : nbox_total;  // hot: 2048 boxes of this size cycle through L2
    const int row = (int)((rng >> 4) % (uint32_t)nb) * brows;
    if (store)
      tma_store_2d(&m, smem + (it & 7) * bbytes, 0, row);
    else
      tma_reduce_add_2d(&m, smem + (it & 7) * bbytes, 0, row);
    bulk_commit();
  }
  bulk_wait0();
  out[blockIdx.x] = (unsigned long long)(clock64() - t0);
}

// mixed: warp 0 lane 0 TMA-reduces 4 KB boxes (8 in flight); warps 1..4 issue row-coalesced
// red.global.add.v4 (each instruction 512 B contiguous) into a disjoint region; both for `iters`
__global__ void __launch_bounds__(160, 1) mixed_kernel(const __grid_constant__ CUtensorMap m, float* buf2, size_t n2,
                                                       int iters, int use_tma, int use_red, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long t0 = clock64();
  if (warp == 0) {
    if (lane == 0 && use_tma) {
      for (int i = 0; i < 8 * 4096 / 4; ++i) reinterpret_cast<float*>(smem)[i] = 1.f;
      fence_async_smem();
      uint32_t rng = 777u + blockIdx.x * 7919u;
      for (int it = 0; it < iters; ++it) {
        if (it >= 8) bulk_wait_group_read<7>();
        rng = rng * 1664525u + 1013904223u;
        tma_reduce_add_2d(&m, smem + (it & 7) * 4096, 0, (int)((rng >> 4) % 2048u) * 32);
        bulk_commit();
      }
      bulk_wait0();
    }
  } else if (use_red) {
    uint32_t rng = 99u + blockIdx.x * 131u + warp;
    for (int it = 0; it < iters / 4 * 8; ++it) {  // same bytes as the TMA side per warp-quad: iters*4KB total
      rng = rng * 1664525u + 1013904223u;
      float* dst = buf2 + ((size_t)((rng >> 4) % (uint32_t)(n2 / 128)) * 128) + lane * 4;
      red_add_v4(dst, 1.f, 1.f, 1.f, 1.f);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(clock64() - t0);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const size_t rows = (size_t)8 * 2048 * 32 * 128 / 32;  // 268 MB fp32 as {32, rows}
  float* buf;
  cudaMalloc(&buf, rows * 32 * 4);
  cudaMemset(buf, 0, rows * 32 * 4);
  EncodeFn enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(red_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int brows : {32}) {
    CUtensorMap m;
    cuuint64_t dims[2] = {32, rows};
    cuuint64_t str[1] = {32 * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)brows}, es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int store = 1; store >= 0; --store) {
      for (int hot = 0; hot < 2; ++hot) {
        for (int grid : {1, 148}) {
          const int iters = 2048 * 32 / brows;
          float ms = 0;
          double c = 0;
          for (int w = 0; w < 2; ++w) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            red_kernel<<<grid, 32, 200 * 1024>>>(m, (int)(rows / brows), iters, store, brows, hot, d);
            cudaEventRecord(e1);
            if (cudaEventSynchronize(e1) != cudaSuccess) { printf("err\n"); return 1; }
            cudaEventElapsedTime(&ms, e0, e1);
            std::vector<unsigned long long> h(grid);
            cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
            c = 0;
            for (auto x : h) c += x;
            c /= grid;
          }
          printf("%s box 32x%-3d %s grid %3d: %5.1f B/clk per SM, %5.0f GB/s chip-wide\n",
                 store ? "TMA store     " : "TMA reduce-add", brows, hot ? "L2-hot " : "268 MB ", grid,
                 (double)iters * brows * 128 / c, (double)grid * iters * brows * 128 / ms / 1e6);
        }
      }
    }
  }
  {
    CUtensorMap m;
    cuuint64_t dims[2] = {32, rows};
    cuuint64_t str[1] = {32 * 4};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    float* buf2;
    const size_t n2 = (size_t)2048 * 4096 / 4;  // 8 MB hot region
    cudaMalloc(&buf2, n2 * 4);
    cudaMemset(buf2, 0, n2 * 4);
    cudaFuncSetAttribute(mixed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int mode = 1; mode <= 3; ++mode) {
      const int use_tma = mode & 1, use_red = (mode >> 1) & 1, iters = 2048;
      for (int grid : {1, 148}) {
        double c = 0;
        for (int w = 0; w < 2; ++w) {
          mixed_kernel<<<grid, 160, 64 * 1024>>>(m, buf2, n2, iters, use_tma, use_red, d);
          if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
          std::vector<unsigned long long> h(grid);
          cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
          c = 0;
          for (auto x : h) c += x;
          c /= grid;
        }
        const double bytes = (use_tma ? iters * 4096.0 : 0) + (use_red ? iters / 4 * 8 * 512.0 * 4 : 0);
        printf("mixed %s%s grid %3d: %.1f B/clk per SM total\n", use_tma ? "TMA-reduce " : "", use_red ? "LSU-red " : "",
               grid, bytes / c);
      }
    }
  }
  return 0;
}
