// mma_bench.cu — tcgen05.mma issue-rate microbenchmark for the operand layouts used
// by the conv kernels (SS mode, kind::f16, M = 128, cta_group::1).
// One CTA per SM, one thread issues R back-to-back MMAs into TMEM with fixed
// descriptors; reports cycles per MMA and the fraction of the dense floor
// 128*N/256 cycles (B300_MICROARCH.md "tcgen05 floor").
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../paper_2207_01053_b200/csrc tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "tc.cuh"

using namespace protea;

struct Cfg {
  const char* name;
  int N;
  bool a_mn, b_mn;
  int a_layout, b_layout;  // 0 none, 4 sw64, 2 sw128
  uint32_t a_lbo, a_sbo, b_lbo, b_sbo;
  uint32_t a_kstep, b_kstep;  // start-address advance per MMA (cycled over 8 steps)
};

__device__ uint64_t mkdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, int layout) {
  uint64_t d = tc::sdesc(addr, lbo, sbo);
  return d | ((uint64_t)layout << 61);
}

__global__ void __launch_bounds__(128, 1) k_mma_bench(Cfg c, int R, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    tc::mbar_init(tc::smem_u32(&bar), 1);
    tc::mbar_fence_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(tc::smem_u32(&slot), 512);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t sa = tc::smem_u32(smem), sb = sa + 64 * 1024;
    const uint32_t idesc = tc::idesc_bf16(128, c.N, c.a_mn, c.b_mn);
    const long long t0 = clock64();
    for (int i = 0; i < R; ++i) {
      const int k = i & 7;
      tc::mma_bf16(tmem, mkdesc(sa + k * c.a_kstep, c.a_lbo, c.a_sbo, c.a_layout),
                   mkdesc(sb + k * c.b_kstep, c.b_lbo, c.b_sbo, c.b_layout), idesc, 1);
    }
    tc::commit(tc::smem_u32(&bar));
    tc::mbar_wait(tc::smem_u32(&bar), 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

__device__ __forceinline__ void mma_elect(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_elect(uint32_t mbar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(mbar)
      : "memory");
}

// variant: descriptors precomputed (8 per operand), 8-way unrolled; mode 0 = thread 0 only, 1 = warp 0 + elect.sync
__global__ void __launch_bounds__(128, 1) k_mma_bench2(Cfg c, int R, int mode, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    tc::mbar_init(tc::smem_u32(&bar), 1);
    tc::mbar_fence_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(tc::smem_u32(&slot), 512);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = slot;
  const uint32_t sa = tc::smem_u32(smem), sb = sa + 64 * 1024;
  const uint32_t idesc = tc::idesc_bf16(128, c.N, c.a_mn, c.b_mn);
  uint64_t da[8], db[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    da[k] = mkdesc(sa + k * c.a_kstep, c.a_lbo, c.a_sbo, c.a_layout);
    db[k] = mkdesc(sb + k * c.b_kstep, c.b_lbo, c.b_sbo, c.b_layout);
  }
  if (mode == 0 && threadIdx.x == 0) {
    const long long t0 = clock64();
    for (int i = 0; i < R; i += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) tc::mma_bf16(tmem, da[k], db[k], idesc, 1);
    }
    tc::commit(tc::smem_u32(&bar));
    tc::mbar_wait(tc::smem_u32(&bar), 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
  } else if (mode == 1 && threadIdx.x < 32) {
    const long long t0 = clock64();
    for (int i = 0; i < R; i += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) mma_elect(tmem, da[k], db[k], idesc, 1);
    }
    commit_elect(tc::smem_u32(&bar));
    tc::mbar_wait(tc::smem_u32(&bar), 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

int main() {
  // K-major SW128: atom 8 rows x 128 B, SBO 1024, k-step +32 B.  K-major none: core matrices
  // [rows/8][2][128 B] -> LBO 128 (k), SBO 256 (m).  MN-major none: LBO = k-group stride, SBO = 128.
  Cfg cfgs[] = {
      {"Kmaj SW128 A / Kmaj SW128 B  N=64 ", 64, false, false, 2, 2, 16, 1024, 16, 1024, 32, 32},
      {"Kmaj SW128 A / Kmaj SW128 B  N=128", 128, false, false, 2, 2, 16, 1024, 16, 1024, 32, 32},
      {"Kmaj SW128 A / Kmaj SW128 B  N=256", 256, false, false, 2, 2, 16, 1024, 16, 1024, 32, 32},
      {"Kmaj SW128 A / Kmaj SW128 B  N=48 ", 48, false, false, 2, 2, 16, 1024, 16, 1024, 32, 32},
      {"Kmaj none  A / Kmaj none  B  N=64 ", 64, false, false, 0, 0, 128, 256, 128, 256, 4096, 4096},
      {"Kmaj none  A / Kmaj none  B  N=128", 128, false, false, 0, 0, 128, 256, 128, 256, 4096, 4096},
      {"Kmaj none  A / Kmaj none  B  N=256", 256, false, false, 0, 0, 128, 256, 128, 256, 4096, 4096},
      {"Kmaj SW64  A / Kmaj none  B  N=64 ", 64, false, false, 4, 0, 16, 512, 128, 256, 32, 4096},
      {"Kmaj none  A(LBO160,SBO640) / Kmaj none B N=128", 128, false, false, 0, 0, 160, 640, 2048, 128, 16, 4096},
      {"MN SW128 A / MN none B  N=48 (wgrad)", 48, true, true, 2, 0, 16384, 1024, 256, 4608, 2048, 128},
      {"MN SW128 A / MN none B  N=144", 144, true, true, 2, 0, 16384, 1024, 4608, 128, 2048, 128},
      {"MN SW128 A / MN SW128 B N=64 ", 64, true, true, 2, 2, 16384, 1024, 8192, 1024, 2048, 2048},
      {"MN SW128 A / MN SW128 B N=128", 128, true, true, 2, 2, 16384, 1024, 8192, 1024, 2048, 2048},
      {"MN none A / MN none B N=64", 64, true, true, 0, 0, 2048, 128, 1024, 128, 4096, 2048},
      {"MN SW64 A(LBO1024) / MN SW128 B N=64 (c2 wgrad)", 64, true, true, 4, 2, 1024, 512, 16, 1024, 1024, 2048},
      {"MN SW64 A(LBO12288) / MN SW128 B N=64", 64, true, true, 4, 2, 12288, 512, 16, 1024, 1024, 2048},
      {"MN SW64 A(LBO4096) / MN SW128 B N=64", 64, true, true, 4, 2, 4096, 512, 16, 1024, 1024, 2048},
      {"Kmaj SW64 A(SBO512) / MN none B N=32 (c2 dgrad-ish)", 32, false, true, 4, 0, 16, 512, 128, 512, 32, 256},
      {"Kmaj SW128 A / Kmaj SW128 B N=32", 32, false, false, 2, 2, 16, 1024, 16, 1024, 32, 32},
      {"Kmaj SW128 A / Kmaj SW128 B N=16", 16, false, false, 2, 2, 16, 1024, 16, 1024, 32, 32},
  };
  cudaFuncSetAttribute(k_mma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 161 * 1024);
  cudaFuncSetAttribute(k_mma_bench2, cudaFuncAttributeMaxDynamicSharedMemorySize, 161 * 1024);
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int R = 8192;
  for (const Cfg& c : cfgs) {
    for (int grid : {148}) {
      k_mma_bench<<<grid, 128, 161 * 1024>>>(c, R, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long cy = 0;
      cudaMemcpy(&cy, d, 8, cudaMemcpyDeviceToHost);
      const double per = (double)cy / R, floor = 128.0 * c.N / 256.0;
      printf("%-48s grid %3d: %7.2f cyc/mma  floor %6.1f  eff %5.1f%%  %s\n", c.name, grid, per, floor,
             100.0 * floor / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    for (int mode = 0; mode < 2; ++mode) {
      k_mma_bench2<<<148, 128, 161 * 1024>>>(c, R, mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long cy = 0;
      cudaMemcpy(&cy, d, 8, cudaMemcpyDeviceToHost);
      const double per = (double)cy / R, floor = 128.0 * c.N / 256.0;
      printf("%-48s %s: %7.2f cyc/mma  floor %6.1f  eff %5.1f%%  %s\n", c.name, mode ? "elect " : "unroll", per,
             floor, 100.0 * floor / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
