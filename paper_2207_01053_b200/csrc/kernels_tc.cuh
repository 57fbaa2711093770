// kernels_tc.cuh — bf16 tensor-core (tcgen05 / TMEM) grouped GEMMs of one
// lock-step iteration (bf16 mode).
//
// Same grouped structure as kernels_simt.cuh (one launch per layer-op over every
// active client; CTA -> (client, tile) by binary search over a prefix table),
// but each CTA computes a 128 x BN output tile on the 5th-generation tensor
// cores: 4 producer warps stream 64-wide K blocks of both operands into a
// STAGES-deep shared-memory ring with 16-byte cp.async (the operands are
// implicit-GEMM gathers: im2col of NHWC activations, transposed weights, ...),
// one elected thread of warp 4 issues tcgen05.mma (M=128, N=BN, K=16, bf16 in,
// fp32 accumulate in TMEM) and tcgen05.commit releases each stage, and the 4
// producer warps then drain the accumulator with tcgen05.ld and run the
// layer's fused epilogue (bias+ReLU+2x2 pool / ReLU-mask + pool-backward
// scatter / SGD update of fp32 master + bf16 shadow weights).
//
// Op sizes per client-step (rows = |beta|, CNN-w channels c1, c2, F; K1 = 64 c2):
//   conv2 fwd   M = rows*256 (quad-major) N = c2    K = 25 c1      A K-major, B K-major
//   conv2 dgrad M = rows*256              N = c1    K = 25 c2      A K-major, B MN-major
//   conv2 wgrad M = 25 c1 + 1 (bias row)  N = c2    K = rows*256   A MN-major, B MN-major
//   fc1 fwd     M = F                     N = rows  K = K1         A K-major, B K-major
//   fc1 dgrad   M = K1                    N = rows  K = F          A MN-major, B K-major
//   fc1 wgrad   M = K1                    N = F     K = rows       A MN-major, B MN-major
#pragma once
#include "device.cuh"
#include "kernels_simt.cuh"
#include "tc.cuh"

namespace protea {

typedef __nv_bfloat16 bf16;

struct TcTile {
  const ClientRec* c;
  Task tk;
  int m0, n0;
  int nk;     // 64-wide K blocks
  int n_mma;  // instruction N (multiple of 16, <= BN)
};

__device__ __align__(16) const uint16_t kOneChunk[8] = {0x3F80, 0, 0, 0, 0, 0, 0, 0};  // bf16 {1,0,...,0}

template <bool MN, int R>
__device__ __forceinline__ void chunk_coords(int q, int& i, int& j) {
  if (MN) {  // i = k row in [0,64), j = mn group in [0, R/8)
    i = (q / R) * 8 + (q & 7);
    j = (q >> 3) % (R / 8);
  } else {  // i = mn row in [0, R), j = k chunk in [0, 8)
    i = (q >> 6) * 8 + (q & 7);
    j = (q >> 3) & 7;
  }
}

constexpr int kTcThreads = 160;

template <int BN, int STAGES>
constexpr int tc_smem_bytes() {
  return STAGES * (128 * 64 * 2 + BN * 64 * 2) + (2 * STAGES + 1) * 8 + 16;
}

template <int BN, int STAGES, class Op>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_gemm_tc(const Op op, const Task* __restrict__ tasks, const int* __restrict__ prefix, int ntask) {
  constexpr int A_BYTES = 128 * 64 * 2, B_BYTES = BN * 64 * 2, STAGE = A_BYTES + B_BYTES;
  constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  constexpr int LAG = (STAGES - 1) < 2 ? (STAGES - 1) : 2;
  static_assert(LAG >= 1, "need >= 2 stages");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int ti = find_task(prefix, ntask, blockIdx.x);
  TcTile t;
  t.tk = tasks[ti];
  t.c = op.recs + t.tk.rec;
  op.setup(t, blockIdx.x - __ldg(prefix + ti));

  const uint32_t bar0 = tc::smem_u32(bars);
  const uint32_t done = bar0 + 16 * STAGES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(bar0 + 8 * s, 128);             // full[s]: one arrive per producer thread
      tc::mbar_init(bar0 + 8 * (STAGES + s), 1);    // empty[s]: tcgen05.commit
    }
    tc::mbar_init(done, 1);
    tc::mbar_fence_init();
  }
  if (warp == 4) tc::tmem_alloc(tc::smem_u32(tmem_slot), TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = tc::smem_u32(smem);

  if (warp < 4) {
    // ---------------- producers
    const int tid = threadIdx.x;
    const void* any = op.any(t);
    for (int kb = 0; kb < t.nk; ++kb) {
      const int s = kb % STAGES;
      if (kb >= STAGES) tc::mbar_wait(bar0 + 8 * (STAGES + s), ((kb / STAGES) - 1) & 1);
      const uint32_t a_base = sbase + s * STAGE, b_base = a_base + A_BYTES;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int q = tid + 128 * u;
        int i, j;
        chunk_coords<Op::A_MN, 128>(q, i, j);
        tc::cp16(a_base + 16 * q, op.a_src(t, kb, i, j), any);
      }
#pragma unroll
      for (int u = 0; u < BN * 8 / 128; ++u) {
        const int q = tid + 128 * u;
        int i, j;
        chunk_coords<Op::B_MN, BN>(q, i, j);
        tc::cp16(b_base + 16 * q, op.b_src(t, kb, i, j), any);
      }
      tc::cp_commit();
      if (kb >= LAG) {
        tc::cp_wait<LAG>();
        tc::fence_proxy_async();
        tc::mbar_arrive(bar0 + 8 * ((kb - LAG) % STAGES));
      }
    }
    tc::cp_wait<0>();
    tc::fence_proxy_async();
    for (int kb = (t.nk - LAG > 0 ? t.nk - LAG : 0); kb < t.nk; ++kb) tc::mbar_arrive(bar0 + 8 * (kb % STAGES));

    // ---------------- epilogue: TMEM -> registers -> fused layer epilogue
    tc::mbar_wait(done, 0);
    tc::fence_after();
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < t.n_mma; c0 += 16) {
      float v[16];
      tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
      op.epilogue(t, row, c0, v);
    }
  } else if (warp == 4) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_bf16(128, t.n_mma, Op::A_MN, Op::B_MN);
      for (int kb = 0; kb < t.nk; ++kb) {
        const int s = kb % STAGES;
        tc::mbar_wait(bar0 + 8 * s, (kb / STAGES) & 1);
        tc::fence_after();
        const uint32_t a_base = sbase + s * STAGE, b_base = a_base + A_BYTES;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t da = Op::A_MN ? tc::sdesc(a_base + 32 * 128 * ks, 16 * 128, 128)
                                       : tc::sdesc(a_base + 256 * ks, 128, 1024);
          const uint64_t db = Op::B_MN ? tc::sdesc(b_base + 32 * BN * ks, 16 * BN, 128)
                                       : tc::sdesc(b_base + 256 * ks, 128, 1024);
          tc::mma_bf16(tmem, da, db, idesc, (kb | ks) != 0);
        }
        tc::commit(bar0 + 8 * (STAGES + s));
      }
      tc::commit(done);
    }
    __syncwarp();
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 4) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, TMEM_COLS);
  }
}

__device__ __forceinline__ int round16(int x) { return (x + 15) & ~15; }

// --------------------------------------------------------------------------
// CNN ops on tensor cores (bf16 activations, bf16 shadow weights B_WSH)
// --------------------------------------------------------------------------
struct TcConv2Fwd {
  static constexpr bool A_MN = false, B_MN = false;
  const ClientRec* recs;
  CnnDims d;
  __device__ void setup(TcTile& t, int local) const {
    t.m0 = local * 128;
    t.n0 = 0;
    t.nk = cdiv(25 * d.c1, 64);
    t.n_mma = round16(d.c2);
  }
  __device__ const void* any(const TcTile& t) const { return t.c->params; }
  __device__ const void* a_src(const TcTile& t, int kb, int i, int j) const {
    const int k = kb * 64 + 8 * j;
    if (k >= 25 * d.c1) return nullptr;
    const int m = t.m0 + i, r = m >> 8, local = m & 255, p = local >> 2, q = local & 3;
    const int y = ((p >> 3) << 1) + (q >> 1), x = ((p & 7) << 1) + (q & 1);
    const int tap = k / d.c1, ci = k - tap * d.c1, ky = tap / 5, kx = tap - ky * 5;
    const int sy = y + ky - 2, sx = x + kx - 2;
    if ((unsigned)sy >= 16u || (unsigned)sx >= 16u) return nullptr;
    return (const bf16*)t.c->buf[B_A1] + ((int64_t)r * 256 + sy * 16 + sx) * d.c1 + ci;
  }
  __device__ const void* b_src(const TcTile& t, int kb, int i, int j) const {
    const int k = kb * 64 + 8 * j;
    if (k >= 25 * d.c1 || i >= d.c2) return nullptr;
    return (const bf16*)t.c->buf[B_WSH] + d.w2 + (int64_t)i * 25 * d.c1 + k;
  }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
    const int m = t.m0 + row, r = m >> 8, p = (m & 255) >> 2, q = m & 3;
    const int base = (threadIdx.x & 31) & ~3;
    bf16* a2 = (bf16*)t.c->buf[B_A2];
    uint8_t* i2 = (uint8_t*)t.c->buf[B_I2];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int n = c0 + j;
      const float val = n < d.c2 ? fmaxf(v[j] + t.c->params[d.b2 + n], 0.f) : 0.f;
      const float v0 = __shfl_sync(0xffffffffu, val, base), v1 = __shfl_sync(0xffffffffu, val, base + 1);
      const float v2 = __shfl_sync(0xffffffffu, val, base + 2), v3 = __shfl_sync(0xffffffffu, val, base + 3);
      if (q == 0 && n < d.c2) {
        float best = v0;
        int arg = 0;
        if (v1 > best) { best = v1; arg = 1; }
        if (v2 > best) { best = v2; arg = 2; }
        if (v3 > best) { best = v3; arg = 3; }
        const int64_t o = ((int64_t)r * 64 + p) * d.c2 + n;
        a2[o] = __float2bfloat16_rn(best);
        i2[o] = (uint8_t)arg;
      }
    }
  }
};

struct TcConv2Dgrad {
  static constexpr bool A_MN = false, B_MN = true;
  const ClientRec* recs;
  CnnDims d;
  __device__ void setup(TcTile& t, int local) const {
    t.m0 = local * 128;
    t.n0 = 0;
    t.nk = cdiv(25 * d.c2, 64);
    t.n_mma = round16(d.c1);
  }
  __device__ const void* any(const TcTile& t) const { return t.c->params; }
  __device__ const void* a_src(const TcTile& t, int kb, int i, int j) const {
    const int k = kb * 64 + 8 * j;
    if (k >= 25 * d.c2) return nullptr;
    const int m = t.m0 + i, r = m >> 8, y = (m >> 4) & 15, x = m & 15;
    const int tap = k / d.c2, co = k - tap * d.c2, ky = tap / 5, kx = tap - ky * 5;
    const int sy = y - ky + 2, sx = x - kx + 2;
    if ((unsigned)sy >= 16u || (unsigned)sx >= 16u) return nullptr;
    return (const bf16*)t.c->buf[B_DZ2] + ((int64_t)r * 256 + sy * 16 + sx) * d.c2 + co;
  }
  __device__ const void* b_src(const TcTile& t, int kb, int i, int j) const {
    const int k = kb * 64 + i, n0 = 8 * j;
    if (k >= 25 * d.c2 || n0 >= d.c1) return nullptr;
    const int tap = k / d.c2, co = k - tap * d.c2;
    return (const bf16*)t.c->buf[B_WSH] + d.w2 + ((int64_t)co * 25 + tap) * d.c1 + n0;
  }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
    const int m = t.m0 + row, r = m >> 8, y = (m >> 4) & 15, x = m & 15;
    const bf16* a1 = (const bf16*)t.c->buf[B_A1];
    const uint8_t* i1 = (const uint8_t*)t.c->buf[B_I1];
    bf16* dz1 = (bf16*)t.c->buf[B_DZC1];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int n = c0 + j;
      if (n >= d.c1) continue;
      const int64_t o = (int64_t)m * d.c1 + n;
      const float val = __bfloat162float(a1[o]) > 0.f ? v[j] : 0.f;
      const int arg = i1[o];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int Y = 2 * y + (q >> 1), X = 2 * x + (q & 1);
        dz1[((int64_t)r * 1024 + Y * 32 + X) * d.c1 + n] = __float2bfloat16_rn(q == arg ? val : 0.f);
      }
    }
  }
};

struct TcConv2Wgrad {  // full reduction in one CTA -> SGD update in the epilogue (no split-K partials)
  static constexpr bool A_MN = true, B_MN = true;
  const ClientRec* recs;
  CnnDims d;
  float lr;
  __device__ void setup(TcTile& t, int local) const {
    t.m0 = local * 128;
    t.n0 = 0;
    t.nk = t.tk.rows * 4;  // rows*256 pixels / 64
    t.n_mma = round16(d.c2);
  }
  __device__ const void* any(const TcTile& t) const { return t.c->params; }
  __device__ const void* a_src(const TcTile& t, int kb, int i, int j) const {
    const int p = kb * 64 + i, mg = t.m0 + 8 * j, Kw = 25 * d.c1;
    if (mg == Kw) return kOneChunk;  // bias row: db = sum_p dz
    if (mg > Kw) return nullptr;
    const int r = p >> 8, y = (p >> 4) & 15, x = p & 15;
    const int tap = mg / d.c1, ci = mg - tap * d.c1, ky = tap / 5, kx = tap - ky * 5;
    const int sy = y + ky - 2, sx = x + kx - 2;
    if ((unsigned)sy >= 16u || (unsigned)sx >= 16u) return nullptr;
    return (const bf16*)t.c->buf[B_A1] + ((int64_t)r * 256 + sy * 16 + sx) * d.c1 + ci;
  }
  __device__ const void* b_src(const TcTile& t, int kb, int i, int j) const {
    const int p = kb * 64 + i, n0 = 8 * j;
    if (n0 >= d.c2) return nullptr;
    return (const bf16*)t.c->buf[B_DZ2] + (int64_t)p * d.c2 + n0;
  }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
    const int m = t.m0 + row, Kw = 25 * d.c1;
    if (m > Kw) return;
    float* P = t.c->params;
    bf16* S = (bf16*)t.c->buf[B_WSH];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int co = c0 + j;
      if (co >= d.c2) continue;
      if (m < Kw) {
        const int64_t idx = d.w2 + (int64_t)co * Kw + m;
        const float w = P[idx] - lr * v[j];
        P[idx] = w;
        S[idx] = __float2bfloat16_rn(w);
      } else {
        P[d.b2 + co] -= lr * v[j];
      }
    }
  }
};

struct TcFc1Fwd {
  static constexpr bool A_MN = false, B_MN = false;
  const ClientRec* recs;
  CnnDims d;
  __device__ void setup(TcTile& t, int local) const {
    t.m0 = local * 128;
    t.n0 = 0;
    t.nk = d.c2;  // 64 c2 / 64
    t.n_mma = round16(t.tk.rows);
  }
  __device__ const void* any(const TcTile& t) const { return t.c->params; }
  __device__ const void* a_src(const TcTile& t, int kb, int i, int j) const {
    return (const bf16*)t.c->buf[B_WSH] + d.w3 + (int64_t)(t.m0 + i) * 64 * d.c2 + kb * 64 + 8 * j;
  }
  __device__ const void* b_src(const TcTile& t, int kb, int i, int j) const {
    if (i >= t.tk.rows) return nullptr;
    return (const bf16*)t.c->buf[B_A2] + (int64_t)i * 64 * d.c2 + kb * 64 + 8 * j;
  }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
    const int f = t.m0 + row;
    const float b = t.c->params[d.b3 + f];
    bf16* h = (bf16*)t.c->buf[B_H];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int r = c0 + j;
      if (r < t.tk.rows) h[(int64_t)r * d.f + f] = __float2bfloat16_rn(fmaxf(v[j] + b, 0.f));
    }
  }
};

struct TcFc1Dgrad {
  static constexpr bool A_MN = true, B_MN = false;
  const ClientRec* recs;
  CnnDims d;
  __device__ void setup(TcTile& t, int local) const {
    t.m0 = local * 128;
    t.n0 = 0;
    t.nk = d.f / 64;
    t.n_mma = round16(t.tk.rows);
  }
  __device__ const void* any(const TcTile& t) const { return t.c->params; }
  __device__ const void* a_src(const TcTile& t, int kb, int i, int j) const {
    const int f = kb * 64 + i;
    return (const bf16*)t.c->buf[B_WSH] + d.w3 + (int64_t)f * 64 * d.c2 + t.m0 + 8 * j;
  }
  __device__ const void* b_src(const TcTile& t, int kb, int i, int j) const {
    if (i >= t.tk.rows) return nullptr;
    return (const bf16*)t.c->buf[B_DH] + (int64_t)i * d.f + kb * 64 + 8 * j;
  }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
    const int n1 = t.m0 + row, K1 = 64 * d.c2;
    const int p = n1 / d.c2, c = n1 - p * d.c2, py = p >> 3, px = p & 7;
    const bf16* a2 = (const bf16*)t.c->buf[B_A2];
    const uint8_t* i2 = (const uint8_t*)t.c->buf[B_I2];
    bf16* dz2 = (bf16*)t.c->buf[B_DZ2];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int r = c0 + j;
      if (r >= t.tk.rows) continue;
      const int64_t o = (int64_t)r * K1 + n1;
      const float val = __bfloat162float(a2[o]) > 0.f ? v[j] : 0.f;
      const int arg = i2[o];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int y = 2 * py + (q >> 1), x = 2 * px + (q & 1);
        dz2[((int64_t)r * 256 + y * 16 + x) * d.c2 + c] = __float2bfloat16_rn(q == arg ? val : 0.f);
      }
    }
  }
};

struct TcFc1Wgrad {  // M = K1 (input features), N = F (outputs), K = rows; W <- W - lr dW
  static constexpr bool A_MN = true, B_MN = true;
  const ClientRec* recs;
  CnnDims d;
  float lr;
  __device__ void setup(TcTile& t, int local) const {
    const int nt = cdiv(d.f, 256);
    t.m0 = (local / nt) * 128;
    t.n0 = (local % nt) * 256;
    t.nk = 1;  // rows <= 64
    t.n_mma = min(256, d.f - t.n0);
  }
  __device__ const void* any(const TcTile& t) const { return t.c->params; }
  __device__ const void* a_src(const TcTile& t, int kb, int i, int j) const {
    if (i >= t.tk.rows) return nullptr;
    return (const bf16*)t.c->buf[B_A2] + (int64_t)i * 64 * d.c2 + t.m0 + 8 * j;
  }
  __device__ const void* b_src(const TcTile& t, int kb, int i, int j) const {
    const int n = t.n0 + 8 * j;
    if (i >= t.tk.rows || n >= d.f) return nullptr;
    return (const bf16*)t.c->buf[B_DH] + (int64_t)i * d.f + n;
  }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
    const int k1 = t.m0 + row, K1 = 64 * d.c2;
    float* P = t.c->params;
    bf16* S = (bf16*)t.c->buf[B_WSH];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int f = t.n0 + c0 + j;
      if (f >= d.f) continue;
      const int64_t idx = d.w3 + (int64_t)f * K1 + k1;
      const float w = P[idx] - lr * v[j];
      P[idx] = w;
      S[idx] = __float2bfloat16_rn(w);
    }
  }
};

// --------------------------------------------------------------------------
// self-test GEMM (protea_selftest_gemm): D[M,N] = A B^T with dense bf16 operands
// --------------------------------------------------------------------------
struct TcDense {
  // A: K-major [M][K] (a_mn=0) or MN-major [K][M]; B likewise with N; K multiple of 64; M multiple of 128
  static constexpr bool A_MN = false, B_MN = false;
  const ClientRec* recs;
  const bf16* A;
  const bf16* B;
  float* D;
  int M, N, K;
  __device__ void setup(TcTile& t, int local) const {
    t.m0 = local * 128;
    t.n0 = 0;
    t.nk = K / 64;
    t.n_mma = round16(N);
  }
  __device__ const void* any(const TcTile& t) const { return A; }
  __device__ const void* a_src(const TcTile& t, int kb, int i, int j) const {
    return A + (int64_t)(t.m0 + i) * K + kb * 64 + 8 * j;
  }
  __device__ const void* b_src(const TcTile& t, int kb, int i, int j) const {
    if (i >= N) return nullptr;
    return B + (int64_t)i * K + kb * 64 + 8 * j;
  }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (c0 + j < N) D[(int64_t)(t.m0 + row) * N + c0 + j] = v[j];
  }
};

struct TcDenseMN {  // A given as [K][M] (MN-major), B as [K][N] (MN-major)
  static constexpr bool A_MN = true, B_MN = true;
  const ClientRec* recs;
  const bf16* A;
  const bf16* B;
  float* D;
  int M, N, K;
  __device__ void setup(TcTile& t, int local) const {
    t.m0 = local * 128;
    t.n0 = 0;
    t.nk = K / 64;
    t.n_mma = round16(N);
  }
  __device__ const void* any(const TcTile& t) const { return A; }
  __device__ const void* a_src(const TcTile& t, int kb, int i, int j) const {
    return A + (int64_t)(kb * 64 + i) * M + t.m0 + 8 * j;
  }
  __device__ const void* b_src(const TcTile& t, int kb, int i, int j) const {
    if (8 * j >= N) return nullptr;
    return B + (int64_t)(kb * 64 + i) * N + 8 * j;
  }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (c0 + j < N) D[(int64_t)(t.m0 + row) * N + c0 + j] = v[j];
  }
};

}  // namespace protea
