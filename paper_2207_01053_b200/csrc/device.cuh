// device.cuh — device-side records and small helpers shared by all kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.h"

namespace protea {

// One client of the round on this rank (device copy; built on host per round).
struct ClientRec {
  float* params;           // P fp32 master weights in the slot
  int32_t* perm;           // E*n epoch permutations
  float* stats;            // 16 floats: [0] loss sum
  void* buf[B_COUNT];      // slot buffers (nullptr if unused)
  const uint8_t* x;        // device shard, n x D u8
  const int32_t* y;        // labels
  const float* wg;         // global weights of the client's group (device)
  double* acc;             // group FedAvg accumulator (fp64)
  int32_t n, B, E, nb;     // B = min(B_k, n): rows one batch can hold (per-row buffer capacity); nb = ceil(n/B_k)
  int64_t P;               // parameters of the client's model
  int32_t c1;              // CNN conv1 channels (padded conv1 shadow in bf16 mode), else 0
  int32_t pad_;
  int64_t id;
  uint64_t* sm_ns;         // per-client device-time attribution (nullable)
  const void* tmaps;       // bf16 CNN / ResNet-8: kTmapSlots CUtensorMaps (128 B each, global memory), else nullptr
  float* mw;               // micro-client 0 of a batch > kMicroRows: the merge weights (P fp32), else nullptr
  // fp32 master weights of a [F][K] matrix at [sp_off, sp_off + sp_len) (sp_len = F K, sp_k = K, K a multiple
  // of 128) stored as 16-bit halves (bf16-mode CNN: fc1's W, the HBM-bound weight stream): per row f and
  // 128-wide block of k, 128 upper halves then 128 lower halves (512 contiguous bytes, like the fp32 row
  // segment they replace).  The upper halves are the tensor-core operand of fc1 fwd / dgrad, read by TMA as a
  // [F][K/128][128] tensor with a 512-byte block stride; the fp32 value is exactly (hi << 16 | lo); nothing
  // else stores those weights (DESIGN.md §5 "split planes").
  int64_t sp_off, sp_len;
  int64_t sp_k;
};

__device__ __forceinline__ float split_join(uint16_t hi, uint16_t lo) {
  return __uint_as_float(((uint32_t)hi << 16) | lo);
}
// 16-bit index of the upper half of matrix element i = f K + k (the lower half is 128 further)
__device__ __forceinline__ int64_t split_hi_index(const ClientRec* c, int64_t i) {
  const int64_t f = i / c->sp_k, k = i - f * c->sp_k;
  return f * 2 * c->sp_k + (k >> 7) * 256 + (k & 127);
}
// master weight d of client c (either representation)
__device__ __forceinline__ float master_w(const ClientRec* c, int64_t d) {
  const uint64_t i = (uint64_t)(d - c->sp_off);
  if (i < (uint64_t)c->sp_len) {
    const uint16_t* h = reinterpret_cast<const uint16_t*>(c->params + c->sp_off) + split_hi_index(c, (int64_t)i);
    return split_join(h[0], h[128]);
  }
  return c->params[d];
}
__device__ __forceinline__ void set_master_w(const ClientRec* c, int64_t d, float w) {
  const uint64_t i = (uint64_t)(d - c->sp_off);
  if (i < (uint64_t)c->sp_len) {
    uint16_t* h = reinterpret_cast<uint16_t*>(c->params + c->sp_off) + split_hi_index(c, (int64_t)i);
    const uint32_t u = __float_as_uint(w);
    h[0] = (uint16_t)(u >> 16);
    h[128] = (uint16_t)(u & 0xFFFFu);
    return;
  }
  c->params[d] = w;
}

// One active client in one lock-step iteration.
struct Task {
  int32_t rec;   // ClientRec index
  int32_t den;   // |beta| of the whole batch: the mean-loss denominator (= rows, except for micro-clients,
                 // which hold a share of a larger batch: common.h kMicroRows)
  int32_t rows;  // rows of the batch in this (micro-)client: min(B, n - j*B) or its share
  int32_t base;  // e*n + j*B: index into perm of the batch's first row
};

// CTA -> task: prefix[i] = first CTA of task i, prefix[ntask] = grid size.
__device__ __forceinline__ int find_task(const int* __restrict__ prefix, int ntask, int block) {
  int lo = 0, hi = ntask - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (__ldg(prefix + mid) <= block)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// Walks a CTA's contiguous tile range task by task; the prefix table is read only
// when the range crosses into the next task (no dependent global load per tile).
struct TaskCursor {
  int ti, lo, hi;  // current task and its tile range [lo, hi)
  __device__ void init(const int* __restrict__ prefix, int ntask, int g) {
    ti = find_task(prefix, ntask, g);
    lo = __ldg(prefix + ti);
    hi = __ldg(prefix + ti + 1);
  }
  __device__ bool advance(const int* __restrict__ prefix, int g) {  // true if the task changed
    if (g < hi) return false;
    do {
      ++ti;
      lo = hi;
      hi = __ldg(prefix + ti + 1);
    } while (g >= hi);
    return true;
  }
};

template <typename T>
__device__ __forceinline__ float ldv(const T* p);
template <>
__device__ __forceinline__ float ldv<float>(const float* p) {
  return *p;
}
template <>
__device__ __forceinline__ float ldv<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}
template <typename T>
__device__ __forceinline__ void stv(T* p, float v);
template <>
__device__ __forceinline__ void stv<float>(float* p, float v) {
  *p = v;
}
template <>
__device__ __forceinline__ void stv<__nv_bfloat16>(__nv_bfloat16* p, float v) {
  *p = __float2bfloat16_rn(v);
}

// u8 pixel -> x/255 (fp32, correctly rounded division)
__device__ __forceinline__ float px01(uint8_t u) { return __fdiv_rn((float)u, 255.0f); }

// SplitMix64 finaliser (reading R10; oracle/splitmix.py is the
// independent Python implementation).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

// Programmatic dependent launch (kernels launched with cudaLaunchAttributeProgrammaticStreamSerialization):
// pdl_wait() blocks until the preceding kernel of the stream has completed and its writes are visible
// (a no-op without the attribute); pdl_trigger() lets the next kernel's CTAs start their prologue.
// Rule used by every kernel of the lock-step chain: all threads call pdl_wait() before touching data the
// preceding kernel may write; only data written two or more kernels earlier (e.g. weights updated in the
// previous step) is read before it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

}  // namespace protea
