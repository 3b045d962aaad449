// Dev microbenchmark: throughput of fp32 global reductions from registers vs plain stores,
// with the access pattern of the diagonal backward pass (one warp instruction = 8 rows x 32 B,
// rows D*4 bytes apart). usage: nvcc -gencode arch=compute_100a,code=sm_100a -O3 red_bw.cu && ./a.out
#include <cstdio>
#include <cuda_runtime.h>

constexpr int D = 128;

template <int MODE>  // 0: st.global.v2.f32, 1: red.global.add.v2.f32, 2: red.global.add.v4.f32
__global__ void k(float* buf, long rows, int reps) {
  const int lane = threadIdx.x & 31, g8 = lane >> 2, c4 = lane & 3;
  const long warps = (long)gridDim.x * (blockDim.x >> 5);
  const long w0 = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (int rep = 0; rep < reps; ++rep)
    for (long rb = w0 * 8; rb < rows; rb += warps * 8) {  // 8 rows per warp item
      float* row = buf + (rb + g8) * D;
#pragma unroll
      for (int dt = 0; dt < D / 8; ++dt) {
        if (MODE == 0) {
          asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(row + dt * 8 + 2 * c4), "f"(1.f), "f"(2.f) : "memory");
        } else if (MODE == 1) {
          asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(row + dt * 8 + 2 * c4), "f"(1.f), "f"(2.f) : "memory");
        } else if (dt % 2 == 0) {
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(row + dt * 8 + 4 * c4), "f"(1.f), "f"(2.f),
                       "f"(3.f), "f"(4.f)
                       : "memory");
        }
      }
    }
}

int main() {
  const long rows = 8L * 2048 * 8 * 12;  // 12 fp32 [B L Hkv D] tensors (dK_i, dV_i, j = 6)
  float* buf;
  cudaMalloc(&buf, rows * D * 4);
  cudaMemset(buf, 0, rows * D * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"st.v2", "red.add.v2", "red.add.v4"};
  for (int mode = 0; mode < 3; ++mode)
    for (int it = 0; it < 3; ++it) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<148 * 4, 256>>>(buf, rows, 1);
      if (mode == 1) k<1><<<148 * 4, 256>>>(buf, rows, 1);
      if (mode == 2) k<2><<<148 * 4, 256>>>(buf, rows, 1);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)rows * D * 4;
      if (it == 2) printf("%-11s %.3f ms  %.2f TB/s of fp32 payload (RMW traffic = 2x)\n", names[mode], ms, bytes / ms / 1e9);
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
