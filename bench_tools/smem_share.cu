// smem_share.cu — dev microbenchmark for the bwd kernel's resource budget:
//  (1) does LSU shared-memory store traffic slow a concurrent SS tcgen05.mma stream
//      (i.e. do they share the 128 B/clk SMEM bandwidth)?
//  (2) throughput of red.global.add.v4.f32 in the dQ-drain pattern (thread = row, 32 x 16 B
//      per thread per 128-column chunk, rows 128 B apart in a tiled fp32 accumulator).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/smem_share bench_tools/smem_share.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2603_18567_b200/csrc/ptx_sm100.cuh"
using namespace tttk;

// warp 0: NI SS MMAs M128 N128 (K-major); warps 1..nst: st.shared.v4 loops over a 32 KB region
__global__ void __launch_bounds__(256, 1) share_kernel(int NI, int nst, int nstore, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  __shared__ volatile int go;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); go = 0; }
  if (warp == 0) { tmem_alloc(&tb, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tb;
  if (warp == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    const uint64_t da = sdesc_sw128(a, 16, 1024), db = sdesc_sw128(b, 16, 1024);
    constexpr uint32_t id = idesc_bf16_f32(128, 128, false, false);
    const long long t0 = clock64();
    for (int i = 0; i < NI; i += 8) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) umma_ss_e(tbase, sdesc_add(da, (ks & 3) * 32), sdesc_add(db, (ks & 3) * 32), id, 1);
    }
    umma_commit_e(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (lane == 0) { out[blockIdx.x * 2] = (unsigned long long)(t1 - t0); go = 1; }
  } else if (warp <= nst) {
    uint8_t* region = smem + 131072 + (warp - 1) * 4096;
    const long long t0 = clock64();
    int n = 0;
    uint4 v = make_uint4(lane, warp, 1, 2);
    while (n < nstore) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(region + lane * 128 + ((k ^ (lane & 7)) << 4))), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
      n += 8;
      v.x += 1;
    }
    const long long t1 = clock64();
    if (lane == 0 && warp == 1) out[blockIdx.x * 2 + 1] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

// (2) 128 threads per CTA; per "tile" each thread adds 32 float4 to its row of a 32-column chunk
__global__ void __launch_bounds__(128) red_kernel(float* acc, size_t tiles_total, int iters, unsigned long long* out) {
  const int row = threadIdx.x;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const size_t tile = (blockIdx.x * 7919ull + it * 104729ull) % tiles_total;
    float* base = acc + tile * 128 * 128;  // [4 chunks][128 rows][32 cols]
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int k = 0; k < 8; ++k)
        red_add_v4(base + ((size_t)c * 128 + row) * 32 + k * 4, 1.f, 1.f, 1.f, 1.f);
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 2 * 8);
  cudaFuncSetAttribute(share_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int NI = 8192;
  for (int nst : {0, 1, 2, 4, 7}) {
    share_kernel<<<148, 256, 200 * 1024>>>(NI, nst, nst ? 20000 : 0, d);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
    std::vector<unsigned long long> h(296);
    cudaMemcpy(h.data(), d, 296 * 8, cudaMemcpyDeviceToHost);
    double m = 0, st = 0;
    for (int i = 0; i < 148; ++i) { m += h[2 * i]; st += h[2 * i + 1]; }
    m /= 148 * (double)NI;
    st /= 148;
    const double st_bytes = nst * 20000.0 * 512;
    printf("MMA SS M128N128 with %d storing warps: %.1f clk/mma (MMA smem %.0f B/clk); stores %.0f B/clk over %.0f clk\n",
           nst, m, 8192.0 / m, nst ? st_bytes / st : 0.0, st);
  }
  // (2)
  const size_t tiles = 4096;  // 4096 tiles x 64 KB = 268 MB (dq_acc size at the Llama shape)
  float* acc;
  cudaMalloc(&acc, tiles * 128 * 128 * 4);
  cudaMemset(acc, 0, tiles * 128 * 128 * 4);
  for (int grid : {148, 296}) {
    const int iters = 64;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    red_kernel<<<grid, 128>>>(acc, tiles, 4, d);
    cudaEventRecord(e0);
    red_kernel<<<grid, 128>>>(acc, tiles, iters, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)grid * iters * 65536;
    std::vector<unsigned long long> h(grid);
    cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
    double c = 0;
    for (auto x : h) c += x;
    c /= grid;
    printf("red.global.add.v4 dQ pattern grid %d: %.1f GB/s of fp32 adds, %.0f clk per 64 KB tile per CTA\n", grid,
           bytes / ms / 1e6, c / iters);
  }
  return 0;
}
