// umma_probe.cu — TEST-ONLY micro-kernels that pin the raw-PTX building blocks
// of the sm_100a path (ptx_sm100.cuh) against a torch matmul, before any
// attention logic depends on them: TMA 128B-swizzle loads, UMMA smem
// descriptors (K-major and MN-major), TMEM accumulators, A-from-TMEM (.kind::f16
// "ts"), manual swizzled smem writes, tcgen05.ld/st, tcgen05.commit.
//
// mode 0: D[m][n] = sum_k A[m][k] B[n][k]        A, B K-major via TMA   (S = Q K^T)
// mode 1: D[m][n] = sum_k P[m][k] V[k][n]        P -> TMEM, V MN-major  (O = P V)
// mode 2: D[m][n] = sum_k X[k][m] Y[k][n]        X manual-swizzled smem as MN-major A,
//                                                 Y via TMA MN-major B   (dQ = dS K)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include "../../paper_2603_18567_b200/csrc/ptx_sm100.cuh"

using namespace tttk;

__global__ void __launch_bounds__(128, 1) probe_kernel(const __grid_constant__ CUtensorMap ma,
                                                       const __grid_constant__ CUtensorMap mb, int mode,
                                                       const __nv_bfloat16* a_glob, float* d) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;              // 32 KB: two [128][64] bf16 boxes
  uint8_t* sB = smem + 32768;      // 32 KB
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(&tmem_base_sh, 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base_sh;
  if (tid == 0) {
    uint32_t bytes = 32768;
    if (mode == 0) {
      bytes += 32768;
      tma_load_4d(sA, &ma, &bar_load, 0, 0, 0, 0);
      tma_load_4d(sA + 16384, &ma, &bar_load, 64, 0, 0, 0);
    }
    tma_load_4d(sB, &mb, &bar_load, 0, 0, 0, 0);
    tma_load_4d(sB + 16384, &mb, &bar_load, 64, 0, 0, 0);
    mbar_expect_tx(&bar_load, bytes);
  }
  if (mode == 1) {
    // thread = row m: pack P[m][0..127] into 64 TMEM columns at tbase + 128
    const __nv_bfloat16* row = a_glob + tid * 128;
    for (int c0 = 0; c0 < 64; c0 += 16) {
      uint32_t r[16];
      for (int i = 0; i < 16; ++i) {
        __nv_bfloat162 v2;
        v2.x = row[2 * (c0 + i)];
        v2.y = row[2 * (c0 + i) + 1];
        r[i] = *reinterpret_cast<uint32_t*>(&v2);
      }
      tmem_st16(tmem_addr(tbase, warp * 32, 128 + c0), r);
    }
    tmem_st_wait();
  } else if (mode == 2) {
    // thread = k row of X[128][128]: write into two [128][64] SW128 boxes
    const __nv_bfloat16* row = a_glob + tid * 128;
    for (int c = 0; c < 128; c += 8) {
      uint4 v = *reinterpret_cast<const uint4*>(row + c);
      const int box = c / 64, cc = c % 64;
      const uint32_t off = box * 16384 + tid * 128 + (((cc / 8) ^ (tid % 8)) * 16);
      *reinterpret_cast<uint4*>(sA + off) = v;
    }
    fence_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    mbar_wait(&bar_load, 0);
    tc_fence_after();
    const uint32_t d_tmem = tbase;  // columns [0,128)
    for (int ks = 0; ks < 8; ++ks) {
      if (mode == 0) {
        const uint32_t ka = smem_u32(sA) + (ks / 4) * 16384 + (ks % 4) * 32;
        const uint32_t kb = smem_u32(sB) + (ks / 4) * 16384 + (ks % 4) * 32;
        umma_ss(d_tmem, sdesc_sw128(ka, 16, 1024), sdesc_sw128(kb, 16, 1024), idesc_bf16_f32(128, 128, false, false),
                ks > 0);
      } else if (mode == 1) {
        const uint32_t kb = smem_u32(sB) + ks * 2048;  // 16 K rows x 128 B
        umma_ts(d_tmem, tmem_addr(tbase, 0, 128 + ks * 8), sdesc_sw128(kb, 16384, 1024),
                idesc_bf16_f32(128, 128, false, true), ks > 0);
      } else {
        const uint32_t ka = smem_u32(sA) + ks * 2048;
        const uint32_t kb = smem_u32(sB) + ks * 2048;
        umma_ss(d_tmem, sdesc_sw128(ka, 16384, 1024), sdesc_sw128(kb, 16384, 1024),
                idesc_bf16_f32(128, 128, true, true), ks > 0);
      }
    }
    umma_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tmem_addr(tbase, warp * 32, c0), r);
    for (int i = 0; i < 32; ++i) d[tid * 128 + c0 + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 256);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static int encode(CUtensorMap* m, const void* ptr) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p) return 1;
  cuuint64_t dims[4] = {128, 1, 128, 1};
  cuuint64_t strides[3] = {256, 256, 128 * 256};
  cuuint32_t box[4] = {64, 1, 128, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return reinterpret_cast<EncodeTiledFn>(p)(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims,
                                            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS;
}

extern "C" int probe_run(int mode, const void* a, const void* b, float* d) {
  CUtensorMap ma, mb;
  if (encode(&ma, a) || encode(&mb, b)) return 1;
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<<<1, 128, smem>>>(ma, mb, mode, reinterpret_cast<const __nv_bfloat16*>(a), d);
  if (cudaGetLastError() != cudaSuccess) return 2;
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 3;
}
