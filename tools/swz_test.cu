// swz_test.cu — does a 64-byte-swizzled UMMA operand tolerate a start address that is
// not a multiple of the 512-byte swizzle atom (a row shift of s x 64 B), and what
// must the descriptor's base-offset field (bits 49-51) hold?  Tests both majors:
//   K-major A  (conv fwd/dgrad halo: rows = pixels, 64 B of K per row)
//   MN-major A (conv2 wgrad: rows = pixels = K, 32 channels = MN per row)
// The A operand is loaded by TMA (CU_TENSOR_MAP_SWIZZLE_64B) exactly like the halos.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_2207_01053_b200/csrc tools/swz_test.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc.cuh"

using namespace protea;

constexpr int R = 160;        // rows (pixels) per A block
constexpr int BLK = R * 64;   // bytes per A block (10 KB, 1024-aligned)

// mode 0: K-major A [m = row][k = 32 ch], 2 K steps; D[m][n] = sum_k A[m+s][k] B[n][k]
// mode 1: MN-major A, 4 blocks of 32 ch at LBO = BLK; K = rows: D[blk*32+c][n] = sum_k A[blk][k+s][c] B[n][k]
__global__ void k_test(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, int mode,
                       int s, int bo, float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t bar, done;
  __shared__ uint32_t slot;
  const uint32_t sa = tc::smem_u32(smem), sbB = sa + 4 * BLK;
  if (threadIdx.x == 0) {
    tc::mbar_init(tc::smem_u32(&bar), 1);
    tc::mbar_init(tc::smem_u32(&done), 1);
    tc::mbar_fence_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(tc::smem_u32(&slot), 32);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    tc::mbar_expect_tx(tc::smem_u32(&bar), 4 * BLK + 16 * 64);
    for (int b = 0; b < 4; ++b) tc::tma_load_2d(sa + b * BLK, &tA, tc::smem_u32(&bar), 0, b * R);
    tc::tma_load_2d(sbB, &tB, tc::smem_u32(&bar), 0, 0);
    tc::mbar_wait(tc::smem_u32(&bar), 0);
    tc::fence_after();
    const uint32_t idesc = tc::idesc_bf16(128, 16, mode == 1, false);
    for (int ks = 0; ks < 2; ++ks) {
      uint64_t da;
      if (mode == 0)
        da = tc::sdesc_sw64(sa + s * 64 + 32 * ks, 16, 512);
      else
        da = tc::sdesc_sw64(sa + s * 64 + 1024 * ks, BLK, 512);
      da |= (uint64_t)(bo & 7) << 49;
      const uint64_t db = tc::sdesc_sw64(sbB + 32 * ks, 16, 512);
      tc::mma_bf16(tmem, da, db, idesc, ks);
    }
    tc::commit(tc::smem_u32(&done));
  }
  __syncwarp();
  tc::mbar_wait(tc::smem_u32(&done), 0);
  tc::fence_after();
  const int row = threadIdx.x;  // 4 warps = 128 lanes
  float v[16];
  tc::tmem_ld16(tmem + ((uint32_t)((threadIdx.x >> 5) * 32) << 16), v);
  for (int n = 0; n < 16; ++n) out[row * 16 + n] = v[n];
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 32);
  }
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

int main() {
  // A: 4 blocks x R rows x 32 ch; B: 16 n x 32 k
  std::vector<__nv_bfloat16> hA(4 * R * 32), hB(16 * 32);
  std::vector<float> fA(hA.size()), fB(hB.size());
  srand(1);
  for (size_t i = 0; i < hA.size(); ++i) { fA[i] = (float)(rand() % 7 - 3); hA[i] = __float2bfloat16(fA[i]); }
  for (size_t i = 0; i < hB.size(); ++i) { fB[i] = (float)(rand() % 5 - 2); hB[i] = __float2bfloat16(fB[i]); }
  void *dA, *dB;
  float* dO;
  cudaMalloc(&dA, hA.size() * 2);
  cudaMalloc(&dB, hB.size() * 2);
  cudaMalloc(&dO, 128 * 16 * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap tA, tB;
  const cuuint64_t dimA[2] = {32, 4 * R}, strA[1] = {64}, dimB[2] = {32, 16}, strB[1] = {64};
  const cuuint32_t boxA[2] = {32, R}, boxB[2] = {32, 16}, es[2] = {1, 1};
  if (cuTensorMapEncodeTiled(&tA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dA, dimA, strA, boxA, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
      cuTensorMapEncodeTiled(&tB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dB, dimB, strB, boxB, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("tensor map encode failed\n");
    return 1;
  }
  const int smem = 4 * BLK + 16 * 64 + 2048;
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<float> o(128 * 16);
  for (int mode = 0; mode < 2; ++mode)
    for (int s : {0, 1, 2, 3, 4, 5, 7, 8, 9}) {
      printf("mode %d (%s) shift %d:", mode, mode ? "MN-major" : "K-major", s);
      for (int bo = 0; bo < 8; ++bo) {
        k_test<<<1, 128, smem>>>(tA, tB, mode, s, bo, dO);
        if (cudaDeviceSynchronize() != cudaSuccess) {
          printf(" bo%d:ERR", bo);
          return 1;
        }
        cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
        double err = 0;
        for (int m = 0; m < 128; ++m)
          for (int n = 0; n < 16; ++n) {
            double ref = 0;
            for (int k = 0; k < 32; ++k) {
              const float a = mode == 0 ? fA[(m + s) * 32 + k] : fA[((m >> 5) * R + k + s) * 32 + (m & 31)];
              ref += (double)a * fB[n * 32 + k];
            }
            err = fmax(err, fabs(ref - o[m * 16 + n]));
          }
        printf(" bo%d:%s", bo, err == 0 ? "OK" : "bad");
      }
      printf("\n");
    }
  return 0;
}
