// tma_lat.cu — dev microbenchmark: latency of one 128-row x 128-col bf16 tile load (two SW128
// boxes of 64 columns) by TMA, as the bwd kernel loads Q: BSHD layout (row stride H*D*2 = 8 KB)
// vs a dense [rows][D] layout (row stride 256 B). One load in flight per CTA; clock64 per load.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/tma_lat bench_tools/tma_lat.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include "../paper_2603_18567_b200/csrc/ptx_sm100.cuh"
using namespace tttk;

__global__ void __launch_bounds__(32, 1) lat_kernel(const __grid_constant__ CUtensorMap m, int ntiles, int nh,
                                                    int nqt, int nb, int inflight, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[4];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
  fence_mbar_init();
  unsigned long long tot = 0;
  uint32_t rng = 12345u + blockIdx.x * 7919u;
  long long t_issue[4];
  auto issue = [&](int s) {
    rng = rng * 1664525u + 1013904223u;
    const int h = (rng >> 8) % nh, qt = (rng >> 16) % nqt, b = (rng >> 4) % nb;
    mbar_expect_tx(&bar[s], 32768);
    t_issue[s] = clock64();
    tma_load_4d(smem + s * 32768, &m, &bar[s], 0, h, qt * 128, b);
    tma_load_4d(smem + s * 32768 + 16384, &m, &bar[s], 64, h, qt * 128, b);
  };
  for (int s = 0; s < inflight; ++s) issue(s);
  for (int i = 0; i < ntiles; ++i) {
    const int s = i % inflight;
    mbar_wait(&bar[s], (i / inflight) & 1);
    tot += clock64() - t_issue[s];
    if (i + inflight < ntiles) issue(s);
  }
  out[blockIdx.x] = tot / ntiles;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int B = 8, L = 2048, H = 32, D = 128;
  void* buf;
  cudaMalloc(&buf, (size_t)B * L * H * D * 2);
  cudaMemset(buf, 0, (size_t)B * L * H * D * 2);
  EncodeFn enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(lat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  for (int layout = 0; layout < 2; ++layout) {
    CUtensorMap m;
    // layout 0: BSHD (D, H, L, B); layout 1: BHSD (D, L-as-dim2 with H folded: dims D, 1->H? use D, L, H, B)
    cuuint64_t dims[4], str[3];
    if (layout == 0) {
      cuuint64_t d4[4] = {(cuuint64_t)D, (cuuint64_t)H, (cuuint64_t)L, (cuuint64_t)B};
      cuuint64_t s3[3] = {(cuuint64_t)D * 2, (cuuint64_t)H * D * 2, (cuuint64_t)L * H * D * 2};
      std::copy(d4, d4 + 4, dims); std::copy(s3, s3 + 3, str);
    } else {  // head-major: row stride 256 B (tile rows contiguous)
      cuuint64_t d4[4] = {(cuuint64_t)D, (cuuint64_t)H, (cuuint64_t)L, (cuuint64_t)B};
      cuuint64_t s3[3] = {(cuuint64_t)L * D * 2, (cuuint64_t)D * 2, (cuuint64_t)L * H * D * 2};
      std::copy(d4, d4 + 4, dims); std::copy(s3, s3 + 3, str);
    }
    cuuint32_t box[4] = {64, 1, 128, 1}, es[4] = {1, 1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    for (int grid : {1, 148}) {
      for (int inflight : {1, 2, 4}) {
        for (int nb : {1, 8}) {  // nb=1: 16 MB working set (L2-resident); nb=8: 134 MB
          lat_kernel<<<grid, 32, 140 * 1024>>>(m, 200, H, L / 128, nb, inflight, d);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
          std::vector<unsigned long long> h(grid);
          cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
          double s = 0;
          for (auto x : h) s += x;
          printf("layout %s grid %3d inflight %d set %s: %.0f clk per 32 KB tile load\n", layout ? "BHSD" : "BSHD", grid,
                 inflight, nb == 1 ? "16MB " : "134MB", s / grid);
        }
      }
    }
  }
  return 0;
}
