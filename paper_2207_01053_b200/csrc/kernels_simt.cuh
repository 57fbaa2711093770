// kernels_simt.cuh — fp32 SIMT kernels of one lock-step iteration (verify path, K8).
//
// Every contraction of local SGD ("finished training"; recipe =
// DESIGN.md reading R10) is written as an implicit GEMM  C[M,N] = sum_k A(m,k) B(k,n)
// over ALL active clients of the iteration at once: the grid is the
// concatenation of every client's tiles (prefix table -> binary search), so
// one launch per layer-op serves the whole cohort ("grouped GEMM").
// Operand loaders and epilogues are per-layer functors:
//   conv fwd    M = pixels (quad-major: 4 consecutive m = one 2x2 pool window),
//               N = cout, K = (ky,kx,ci); epilogue bias + ReLU + 2x2 max-pool
//               (first max wins, strict >) -> pooled value + argmax byte.
//   conv dgrad  M = pixels of the layer input, N = cin, K = (ky,kx,co) (flipped
//               taps); epilogue ReLU mask + pool-backward scatter to full res.
//   conv wgrad  M = cout, N = (ky,kx,ci) + 1 bias column, K = pixels, split-K
//               into fixed chunks; partials summed in split order by k_reduce_update.
//   fc fwd / dgrad / wgrad analogously; fc wgrad applies the SGD update in its
//   epilogue (W <- W - lr dW), after the dgrad kernel read the old W.
// All sums run in a fixed order (deterministic, run-to-run bitwise stable).
#pragma once
#include "device.cuh"

namespace protea {

struct GemmTile {
  const ClientRec* c;
  Task tk;
  int m0, n0, kb, ke, M, N;
  int split;
};

// --------------------------------------------------------------------------
// generic SIMT implicit GEMM
// --------------------------------------------------------------------------
template <int BM, int BN, class Op>
__global__ void __launch_bounds__((BM / 4) * (BN / 4))
    k_gemm_simt(const Op op, const Task* __restrict__ tasks, const int* __restrict__ prefix, int ntask) {
  constexpr int TX = BN / 4, NT = (BM / 4) * (BN / 4), BK = 16;
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN + 4];
  const int ti = find_task(prefix, ntask, blockIdx.x);
  GemmTile t;
  t.tk = tasks[ti];
  t.c = op.recs + t.tk.rec;
  op.setup(t, blockIdx.x - __ldg(prefix + ti));
  const uint64_t t_start = threadIdx.x == 0 ? globaltimer() : 0;
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int k0 = t.kb; k0 < t.ke; k0 += BK) {
    for (int i = tid; i < BM * BK; i += NT) {
      int mm, kk;
      if (Op::A_KFAST) {
        kk = i % BK;
        mm = i / BK;
      } else {
        mm = i % BM;
        kk = i / BM;
      }
      const int m = t.m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < t.M && k < t.ke) ? op.A(t, m, k) : 0.f;
    }
    for (int i = tid; i < BN * BK; i += NT) {
      int nn, kk;
      if (Op::B_KFAST) {
        kk = i % BK;
        nn = i / BK;
      } else {
        nn = i % BN;
        kk = i / BN;
      }
      const int n = t.n0 + nn, k = k0 + kk;
      Bs[kk][nn] = (n < t.N && k < t.ke) ? op.B(t, k, n) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&As[kk][(tid / TX) * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  op.epilogue(t, t.m0 + ty * 4, t.n0 + tx * 4, acc);
  if (threadIdx.x == 0 && t.c->sm_ns)  // K9: per-client SM-time attribution
    atomicAdd((unsigned long long*)t.c->sm_ns, (unsigned long long)(globaltimer() - t_start));
}

// tile decode helpers (host mirrors these in engine.cu: tiles_*())
__host__ __device__ inline int cdiv(int a, int b) { return (a + b - 1) / b; }

// Pool epilogue: thread holds 4 consecutive m (one 2x2 window, q = 2*dy+dx)
// for 4 columns.  relu -> first max (strict >) -> pooled + argmax.
__device__ __forceinline__ void pool4(const float v[4], float& best, int& arg) {
  best = fmaxf(v[0], 0.f);
  arg = 0;
#pragma unroll
  for (int q = 1; q < 4; ++q) {
    const float r = fmaxf(v[q], 0.f);
    if (r > best) {
      best = r;
      arg = q;
    }
  }
}

// --------------------------------------------------------------------------
// CNN-w ops
// --------------------------------------------------------------------------
struct CnnDims {
  int c1, c2, f, classes;
  int64_t w1, b1, w2, b2, w3, b3, w4, b4;  // conv1, conv2, fc1, fc2 offsets in params
  int H, W, C;  // input image (32x32x3 CIFAR-shaped; 28x28x1 FEMNIST-shaped, SIMT kernels only)
  __host__ __device__ int HW() const { return H * W; }                 // conv1 output pixels
  __host__ __device__ int W2() const { return W >> 1; }                // conv2 map width (pool 1)
  __host__ __device__ int HW2() const { return (H >> 1) * (W >> 1); }  // conv2 map pixels
  __host__ __device__ int W4() const { return W >> 2; }                // pool-2 output width
  __host__ __device__ int HW4() const { return (H >> 2) * (W >> 2); }  // pool-2 output pixels
  __host__ __device__ int K1() const { return HW4() * c2; }            // fc1 inputs
};

template <typename T, int BM, int BN>
struct Conv1Fwd {  // M = rows*HW (quad-major over the pooled grid), N = c1, K = 25 C
  static constexpr bool A_KFAST = true, B_KFAST = true;
  const ClientRec* recs;
  CnnDims d;
  __device__ void setup(GemmTile& t, int local) const {
    const int nt = cdiv(d.c1, BN);
    t.M = t.tk.rows * d.HW();
    t.N = d.c1;
    t.m0 = (local / nt) * BM;
    t.n0 = (local % nt) * BN;
    t.kb = 0;
    t.ke = 25 * d.C;
  }
  __device__ float A(const GemmTile& t, int m, int k) const {
    const int HW = d.HW(), r = m / HW, local = m - r * HW, p = local >> 2, q = local & 3;
    const int py = p / d.W2(), px = p - py * d.W2();
    const int y = (py << 1) + (q >> 1), x = (px << 1) + (q & 1);
    const int tap = k / d.C, ci = k - tap * d.C, ky = tap / 5, kx = tap - ky * 5;
    const int sy = y + ky - 2, sx = x + kx - 2;
    if ((unsigned)sy >= (unsigned)d.H || (unsigned)sx >= (unsigned)d.W) return 0.f;
    const int s = t.c->perm[t.tk.base + r];  // sample index of the row's image
    return px01(t.c->x[(int64_t)s * HW * d.C + (sy * d.W + sx) * d.C + ci]);
  }
  __device__ float B(const GemmTile& t, int k, int n) const { return t.c->params[d.w1 + (int64_t)n * 25 * d.C + k]; }
  __device__ void epilogue(const GemmTile& t, int mb, int nb, float acc[4][4]) const {
    if (mb >= t.M) return;
    const int r = mb / d.HW(), p = (mb - r * d.HW()) >> 2;
    T* a1 = (T*)t.c->buf[B_A1];
    uint8_t* i1 = (uint8_t*)t.c->buf[B_I1];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = nb + j;
      if (n >= t.N) continue;
      const float bias = t.c->params[d.b1 + n];
      const float v[4] = {acc[0][j] + bias, acc[1][j] + bias, acc[2][j] + bias, acc[3][j] + bias};
      float best;
      int arg;
      pool4(v, best, arg);
      const int64_t o = ((int64_t)r * d.HW2() + p) * d.c1 + n;
      stv(a1 + o, best);
      i1[o] = (uint8_t)arg;
    }
  }
};

template <typename T, int BM, int BN>
struct Conv2Fwd {  // M = rows*HW2 (quad-major over the pool-2 grid), N = c2, K = 25*c1
  static constexpr bool A_KFAST = true, B_KFAST = true;
  const ClientRec* recs;
  CnnDims d;
  __device__ void setup(GemmTile& t, int local) const {
    const int nt = cdiv(d.c2, BN);
    t.M = t.tk.rows * d.HW2();
    t.N = d.c2;
    t.m0 = (local / nt) * BM;
    t.n0 = (local % nt) * BN;
    t.kb = 0;
    t.ke = 25 * d.c1;
  }
  __device__ float A(const GemmTile& t, int m, int k) const {
    const int HW2 = d.HW2(), W2 = d.W2(), r = m / HW2, local = m - r * HW2, p = local >> 2, q = local & 3;
    const int py = p / d.W4(), px = p - py * d.W4();
    const int y = (py << 1) + (q >> 1), x = (px << 1) + (q & 1);
    const int tap = k / d.c1, ci = k - tap * d.c1, ky = tap / 5, kx = tap - ky * 5;
    const int sy = y + ky - 2, sx = x + kx - 2;
    if ((unsigned)sy >= (unsigned)(d.H >> 1) || (unsigned)sx >= (unsigned)W2) return 0.f;
    const T* a1 = (const T*)t.c->buf[B_A1];
    return ldv(a1 + ((int64_t)r * HW2 + sy * W2 + sx) * d.c1 + ci);
  }
  __device__ float B(const GemmTile& t, int k, int n) const {
    return t.c->params[d.w2 + (int64_t)n * 25 * d.c1 + k];
  }
  __device__ void epilogue(const GemmTile& t, int mb, int nb, float acc[4][4]) const {
    if (mb >= t.M) return;
    const int r = mb / d.HW2(), p = (mb - r * d.HW2()) >> 2;
    T* a2 = (T*)t.c->buf[B_A2];
    uint8_t* i2 = (uint8_t*)t.c->buf[B_I2];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = nb + j;
      if (n >= t.N) continue;
      const float bias = t.c->params[d.b2 + n];
      const float v[4] = {acc[0][j] + bias, acc[1][j] + bias, acc[2][j] + bias, acc[3][j] + bias};
      float best;
      int arg;
      pool4(v, best, arg);
      const int64_t o = ((int64_t)r * d.HW4() + p) * d.c2 + n;
      stv(a2 + o, best);
      i2[o] = (uint8_t)arg;
    }
  }
};

template <typename T, int BM, int BN>
struct Fc1Fwd {  // M = rows, N = f, K = K1 = HW4*c2
  static constexpr bool A_KFAST = true, B_KFAST = true;
  const ClientRec* recs;
  CnnDims d;
  __device__ void setup(GemmTile& t, int local) const {
    const int nt = cdiv(d.f, BN);
    t.M = t.tk.rows;
    t.N = d.f;
    t.m0 = (local / nt) * BM;
    t.n0 = (local % nt) * BN;
    t.kb = 0;
    t.ke = d.K1();
  }
  __device__ float A(const GemmTile& t, int m, int k) const {
    return ldv((const T*)t.c->buf[B_A2] + (int64_t)m * d.K1() + k);
  }
  __device__ float B(const GemmTile& t, int k, int n) const {
    return t.c->params[d.w3 + (int64_t)n * d.K1() + k];
  }
  __device__ void epilogue(const GemmTile& t, int mb, int nb, float acc[4][4]) const {
    T* h = (T*)t.c->buf[B_H];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = mb + i, n = nb + j;
        if (m < t.M && n < t.N) stv(h + (int64_t)m * d.f + n, fmaxf(acc[i][j] + t.c->params[d.b3 + n], 0.f));
      }
  }
};

template <typename T, int BM, int BN>
struct Fc1Dgrad {  // dA2 = dh W1: M = rows, N = K1, K = f; epilogue: pool2 backward -> dz2 (conv2 map)
  static constexpr bool A_KFAST = true, B_KFAST = false;
  const ClientRec* recs;
  CnnDims d;
  __device__ void setup(GemmTile& t, int local) const {
    const int nt = cdiv(d.K1(), BN);
    t.M = t.tk.rows;
    t.N = d.K1();
    t.m0 = (local / nt) * BM;
    t.n0 = (local % nt) * BN;
    t.kb = 0;
    t.ke = d.f;
  }
  __device__ float A(const GemmTile& t, int m, int k) const {
    return ldv((const T*)t.c->buf[B_DH] + (int64_t)m * d.f + k);
  }
  __device__ float B(const GemmTile& t, int k, int n) const {
    return t.c->params[d.w3 + (int64_t)k * d.K1() + n];
  }
  __device__ void epilogue(const GemmTile& t, int mb, int nb, float acc[4][4]) const {
    const T* a2 = (const T*)t.c->buf[B_A2];
    const uint8_t* i2 = (const uint8_t*)t.c->buf[B_I2];
    T* dz2 = (T*)t.c->buf[B_DZ2];
    const int N = t.N;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = mb + i, n = nb + j;
        if (m >= t.M || n >= N) continue;
        const int64_t o = (int64_t)m * N + n;
        const float v = ldv(a2 + o) > 0.f ? acc[i][j] : 0.f;
        const int arg = i2[o];
        const int p = n / d.c2, c = n - p * d.c2, py = p / d.W4(), px = p - py * d.W4();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int y = 2 * py + (q >> 1), x = 2 * px + (q & 1);
          stv(dz2 + ((int64_t)m * d.HW2() + y * d.W2() + x) * d.c2 + c, q == arg ? v : 0.f);
        }
      }
  }
};

template <typename T, int BM, int BN>
struct Fc1Wgrad {  // W1 -= lr dh^T a2: M = f, N = K1, K = rows (fc1 bias: k_head)
  static constexpr bool A_KFAST = false, B_KFAST = false;
  const ClientRec* recs;
  CnnDims d;
  float lr;
  __device__ void setup(GemmTile& t, int local) const {
    const int nt = cdiv(d.K1(), BN);
    t.M = d.f;
    t.N = d.K1();
    t.m0 = (local / nt) * BM;
    t.n0 = (local % nt) * BN;
    t.kb = 0;
    t.ke = t.tk.rows;
  }
  __device__ float A(const GemmTile& t, int m, int k) const {
    return ldv((const T*)t.c->buf[B_DH] + (int64_t)k * d.f + m);
  }
  __device__ float B(const GemmTile& t, int k, int n) const {
    return ldv((const T*)t.c->buf[B_A2] + (int64_t)k * d.K1() + n);
  }
  __device__ void epilogue(const GemmTile& t, int mb, int nb, float acc[4][4]) const {
    const int K1 = d.K1();
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = mb + i, n = nb + j;
        if (m >= t.M || n >= t.N) continue;
        float* w = t.c->params + d.w3 + (int64_t)m * K1 + n;
        *w = *w - lr * acc[i][j];
      }
  }
};

template <typename T, int BM, int BN>
struct Conv2Dgrad {  // dA1: M = rows*HW2 (row-major), N = c1, K = 25*c2; epilogue pool1 backward -> dz1
  static constexpr bool A_KFAST = true, B_KFAST = false;
  const ClientRec* recs;
  CnnDims d;
  __device__ void setup(GemmTile& t, int local) const {
    const int nt = cdiv(d.c1, BN);
    t.M = t.tk.rows * d.HW2();
    t.N = d.c1;
    t.m0 = (local / nt) * BM;
    t.n0 = (local % nt) * BN;
    t.kb = 0;
    t.ke = 25 * d.c2;
  }
  __device__ float A(const GemmTile& t, int m, int k) const {
    const int HW2 = d.HW2(), W2 = d.W2(), r = m / HW2, rem = m - r * HW2, y = rem / W2, x = rem - y * W2;
    const int tap = k / d.c2, co = k - tap * d.c2, ky = tap / 5, kx = tap - ky * 5;
    const int sy = y - ky + 2, sx = x - kx + 2;
    if ((unsigned)sy >= (unsigned)(d.H >> 1) || (unsigned)sx >= (unsigned)W2) return 0.f;
    return ldv((const T*)t.c->buf[B_DZ2] + ((int64_t)r * HW2 + sy * W2 + sx) * d.c2 + co);
  }
  __device__ float B(const GemmTile& t, int k, int n) const {
    const int tap = k / d.c2, co = k - tap * d.c2;
    return t.c->params[d.w2 + ((int64_t)co * 25 + tap) * d.c1 + n];
  }
  __device__ void epilogue(const GemmTile& t, int mb, int nb, float acc[4][4]) const {
    const T* a1 = (const T*)t.c->buf[B_A1];
    const uint8_t* i1 = (const uint8_t*)t.c->buf[B_I1];
    T* dz1 = (T*)t.c->buf[B_DZC1];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = mb + i, n = nb + j;
        if (m >= t.M || n >= t.N) continue;
        const int64_t o = (int64_t)m * d.c1 + n;
        const float v = ldv(a1 + o) > 0.f ? acc[i][j] : 0.f;
        const int arg = i1[o];
        const int HW2 = d.HW2(), W2 = d.W2(), r = m / HW2, rem = m - r * HW2, y = rem / W2, x = rem - y * W2;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int Y = 2 * y + (q >> 1), X = 2 * x + (q & 1);
          stv(dz1 + ((int64_t)r * d.HW() + Y * d.W + X) * d.c1 + n, q == arg ? v : 0.f);
        }
      }
  }
};

// conv wgrad, split-K: partial[split][m][n] for n in [0, N) (N = K_w + 1 bias column)
template <typename T, int BM, int BN>
struct Conv2Wgrad {  // M = c2, N = 25*c1 + 1, K = rows*HW2 pixels (splits of 2048)
  static constexpr bool A_KFAST = false, B_KFAST = false;
  const ClientRec* recs;
  CnnDims d;
  __device__ void setup(GemmTile& t, int local) const {
    const int N = 25 * d.c1 + 1, nt = cdiv(N, BN), mt = cdiv(d.c2, BM);
    t.split = local / (mt * nt);
    const int rem = local - t.split * mt * nt;
    t.M = d.c2;
    t.N = N;
    t.m0 = (rem / nt) * BM;
    t.n0 = (rem % nt) * BN;
    t.kb = t.split * kWgradChunkPx;
    t.ke = min(t.tk.rows * d.HW2(), t.kb + kWgradChunkPx);
  }
  __device__ float A(const GemmTile& t, int m, int k) const {
    return ldv((const T*)t.c->buf[B_DZ2] + (int64_t)k * d.c2 + m);
  }
  __device__ float B(const GemmTile& t, int k, int n) const {
    const int Kw = 25 * d.c1;
    if (n == Kw) return 1.f;
    const int HW2 = d.HW2(), W2 = d.W2(), r = k / HW2, rem = k - r * HW2, y = rem / W2, x = rem - y * W2;
    const int tap = n / d.c1, ci = n - tap * d.c1, ky = tap / 5, kx = tap - ky * 5;
    const int sy = y + ky - 2, sx = x + kx - 2;
    if ((unsigned)sy >= (unsigned)(d.H >> 1) || (unsigned)sx >= (unsigned)W2) return 0.f;
    return ldv((const T*)t.c->buf[B_A1] + ((int64_t)r * HW2 + sy * W2 + sx) * d.c1 + ci);
  }
  __device__ void epilogue(const GemmTile& t, int mb, int nb, float acc[4][4]) const {
    float* part = (float*)t.c->buf[B_WSP] + (int64_t)t.split * t.M * t.N;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = mb + i, n = nb + j;
        if (m < t.M && n < t.N) part[(int64_t)m * t.N + n] = acc[i][j];
      }
  }
};

template <typename T, int BM, int BN>
struct Conv1Wgrad {  // M = c1, N = 25 C + 1, K = rows*HW pixels (splits of 2048)
  static constexpr bool A_KFAST = false, B_KFAST = false;
  const ClientRec* recs;
  CnnDims d;
  __device__ void setup(GemmTile& t, int local) const {
    const int N = 25 * d.C + 1, nt = cdiv(N, BN), mt = cdiv(d.c1, BM);
    t.split = local / (mt * nt);
    const int rem = local - t.split * mt * nt;
    t.M = d.c1;
    t.N = N;
    t.m0 = (rem / nt) * BM;
    t.n0 = (rem % nt) * BN;
    t.kb = t.split * kWgradChunkPx;
    t.ke = min(t.tk.rows * d.HW(), t.kb + kWgradChunkPx);
  }
  __device__ float A(const GemmTile& t, int m, int k) const {
    return ldv((const T*)t.c->buf[B_DZC1] + (int64_t)k * d.c1 + m);
  }
  __device__ float B(const GemmTile& t, int k, int n) const {
    if (n == 25 * d.C) return 1.f;
    const int HW = d.HW(), r = k / HW, rem = k - r * HW, y = rem / d.W, x = rem - y * d.W;
    const int tap = n / d.C, ci = n - tap * d.C, ky = tap / 5, kx = tap - ky * 5;
    const int sy = y + ky - 2, sx = x + kx - 2;
    if ((unsigned)sy >= (unsigned)d.H || (unsigned)sx >= (unsigned)d.W) return 0.f;
    const int s = t.c->perm[t.tk.base + r];
    return px01(t.c->x[(int64_t)s * HW * d.C + (sy * d.W + sx) * d.C + ci]);
  }
  __device__ void epilogue(const GemmTile& t, int mb, int nb, float acc[4][4]) const {
    float* part = (float*)t.c->buf[B_WSP] + (int64_t)t.split * t.M * t.N;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = mb + i, n = nb + j;
        if (m < t.M && n < t.N) part[(int64_t)m * t.N + n] = acc[i][j];
      }
  }
};

// Sum split partials in split order, then W -= lr * g (n < Nw) / b -= lr * g (n == Nw).
struct ReduceArgs {
  const ClientRec* recs;
  int wsp_buf;  // B_WSP or B_R_WSP
  int M, Nw;    // partial is [splits][M][Nw+1]
  int64_t off_w, off_b;
  int px_per_row;  // pixels per sample of the layer output (split count = ceil(rows*px/2048))
  float lr;
  int shadow;      // 1: also write the bf16 weight shadow (bf16 mode); 2: and the padded ResNet conv0 copy
  int layer;       // ResNet-8: the layer's partial region (r8_wsp_off); -1: the buffer start
};
constexpr int kReduceBlock = 256;
__device__ __forceinline__ void reduce_update_block(const ReduceArgs& a, const Task* __restrict__ tasks,
                                                    const int* __restrict__ prefix, int ntask, int block) {
  const int ti = find_task(prefix, ntask, block);
  const Task tk = tasks[ti];
  const ClientRec* c = a.recs + tk.rec;
  const int N = a.Nw + 1, total = a.M * N;
  const int e = (block - prefix[ti]) * kReduceBlock + threadIdx.x;
  if (e >= total) return;
  const int splits = cdiv(tk.rows * a.px_per_row, kWgradChunkPx);
  const float* part = (const float*)c->buf[a.wsp_buf] + (a.layer >= 0 ? r8_wsp_off(a.layer, c->B) : 0);
  float g = 0.f;
  for (int s0 = 0; s0 < splits; s0 += 8) {  // 8 independent loads in flight, summed in split order
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = s0 + j < splits ? __ldcg(part + (int64_t)(s0 + j) * total + e) : 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (s0 + j < splits) g += v[j];
  }
  const int m = e / N, n = e - m * N;
  if (n < a.Nw) {
    const int64_t idx = a.off_w + (int64_t)m * a.Nw + n;
    const float nw = c->params[idx] - a.lr * g;
    c->params[idx] = nw;
    if (a.shadow) ((__nv_bfloat16*)c->buf[B_WSH])[idx] = __float2bfloat16_rn(nw);  // tensor-core operand copy
    if (a.shadow == 2)  // ResNet conv0 (W0 at offset 0, [16][9][3]): the padded [16][9][8] operand copy
      ((__nv_bfloat16*)c->buf[B_R_W0P])[m * 72 + (n / 3) * 8 + n % 3] = __float2bfloat16_rn(nw);
  } else {
    c->params[a.off_b + m] -= a.lr * g;
  }
}

__global__ void __launch_bounds__(kReduceBlock)
    k_reduce_update(ReduceArgs a, const Task* __restrict__ tasks, const int* __restrict__ prefix, int ntask) {
  reduce_update_block(a, tasks, prefix, ntask, blockIdx.x);
}

// ResNet-8: the SGD reduces of all seven conv layers of a step in ONE launch (the layers' partials sit
// in separate regions, r8_wsp_off); block b belongs to layer l with base[l] <= b < base[l + 1].
struct ReduceMulti {
  ReduceArgs a[7];
  const int* prefix[7];
  int base[8];
};
__global__ void __launch_bounds__(kReduceBlock)
    k_reduce_multi(ReduceMulti r, const Task* __restrict__ tasks, int ntask) {
  int l = 0;
  while (l < 6 && (int)blockIdx.x >= r.base[l + 1]) ++l;
  reduce_update_block(r.a[l], tasks, r.prefix[l], ntask, blockIdx.x - r.base[l]);
}

// The same seven reduces with 4 consecutive partial elements per thread (float4 loads; every layer's
// split stride M (Nw + 1) and region offset are multiples of 4 floats) and the client as blockIdx.y
// (every client of a launch has the same layers: no task search).  Block x = (layer l, chunk of
// kReduceBlock * 4 elements) with chunk_base[l] <= x < chunk_base[l + 1].  Per element the splits are
// summed in split order from 0.f exactly as reduce_update_block: bitwise the same update.
struct ReduceMultiV {
  ReduceArgs a[7];
  int chunk_base[8];
};
__global__ void __launch_bounds__(kReduceBlock)
    k_reduce_multi_v4(ReduceMultiV r, const Task* __restrict__ tasks) {
  int l = 0;
  while (l < 6 && (int)blockIdx.x >= r.chunk_base[l + 1]) ++l;
  const ReduceArgs& a = r.a[l];
  const Task tk = tasks[blockIdx.y];
  const ClientRec* c = a.recs + tk.rec;
  const int N = a.Nw + 1, total = a.M * N;
  const int e0 = ((blockIdx.x - r.chunk_base[l]) * kReduceBlock + threadIdx.x) * 4;
  if (e0 >= total) return;
  const int splits = r8_split_cap(a.layer, tk.rows);  // (ResNet-8 only: layer >= 0)
  const float* part = (const float*)c->buf[a.wsp_buf] + r8_wsp_off(a.layer, c->B) + e0;
  float g[4] = {0.f, 0.f, 0.f, 0.f};
  for (int s0 = 0; s0 < splits; s0 += 8) {  // 8 float4 loads in flight
    float4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      v[j] = s0 + j < splits ? __ldcg(reinterpret_cast<const float4*>(part + (int64_t)(s0 + j) * total))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (s0 + j < splits) {
        g[0] += v[j].x;
        g[1] += v[j].y;
        g[2] += v[j].z;
        g[3] += v[j].w;
      }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int e = e0 + k;
    if (e >= total) break;
    const int m = e / N, n = e - m * N;
    if (n < a.Nw) {
      const int64_t idx = a.off_w + (int64_t)m * a.Nw + n;
      const float nw = c->params[idx] - a.lr * g[k];
      c->params[idx] = nw;
      if (a.shadow) ((__nv_bfloat16*)c->buf[B_WSH])[idx] = __float2bfloat16_rn(nw);
      if (a.shadow == 2) ((__nv_bfloat16*)c->buf[B_R_W0P])[m * 72 + (n / 3) * 8 + n % 3] = __float2bfloat16_rn(nw);
    } else {
      c->params[a.off_b + m] -= a.lr * g[k];
    }
  }
}

// --------------------------------------------------------------------------
// MLP ops (784-64-10)
// --------------------------------------------------------------------------
struct MlpDims {
  int classes;
  int64_t w1, b1, w2, b2;
};

template <typename T, int BM, int BN>
struct MlpFc1Fwd {  // M = rows, N = 64, K = 784
  static constexpr bool A_KFAST = true, B_KFAST = true;
  const ClientRec* recs;
  MlpDims d;
  __device__ void setup(GemmTile& t, int local) const {
    const int nt = cdiv(64, BN);
    t.M = t.tk.rows;
    t.N = 64;
    t.m0 = (local / nt) * BM;
    t.n0 = (local % nt) * BN;
    t.kb = 0;
    t.ke = 784;
  }
  __device__ float A(const GemmTile& t, int m, int k) const {
    const int s = t.c->perm[t.tk.base + m];
    return px01(t.c->x[(int64_t)s * 784 + k]);
  }
  __device__ float B(const GemmTile& t, int k, int n) const { return t.c->params[d.w1 + (int64_t)n * 784 + k]; }
  __device__ void epilogue(const GemmTile& t, int mb, int nb, float acc[4][4]) const {
    T* h = (T*)t.c->buf[B_H1];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = mb + i, n = nb + j;
        if (m < t.M && n < t.N) stv(h + (int64_t)m * 64 + n, fmaxf(acc[i][j] + t.c->params[d.b1 + n], 0.f));
      }
  }
};

// MLP fc1 forward for one lock-step iteration: CTA (client, 16 of the 64 outputs).  The rows' u8
// inputs and the CTA's 16 weight rows are staged in shared memory once (the generic tile GEMM
// re-fetched them per 16-wide K step through the permutation: latency-bound at K = 784); every
// thread then runs whole 784-long dot products, accumulated in k order with the same fmaf sequence
// as k_gemm_simt (bitwise-identical h).  Dynamic smem: 16 x 784 fp32 + a 256-entry px01 table + rows x 784 u8.
constexpr int kMlpFwdThreads = 256;
template <typename T>
__global__ void __launch_bounds__(kMlpFwdThreads) k_mlp_fc1_fwd(const ClientRec* __restrict__ recs,
                                                                const Task* __restrict__ tasks, MlpDims d) {
  extern __shared__ __align__(16) uint8_t msm[];
  float* Ws = reinterpret_cast<float*>(msm);  // [16][784]
  float* lut = Ws + 16 * 784;                 // px01(u) for u in [0, 256): the same fp32 values, no division
  uint8_t* xs = msm + (16 * 784 + 256) * 4;   // [rows][784]
  const Task tk = tasks[blockIdx.x];
  const ClientRec* c = recs + tk.rec;
  const int rows = tk.rows, n0 = blockIdx.y * 16;
  const uint64_t t_start = threadIdx.x == 0 ? globaltimer() : 0;
  for (int i = threadIdx.x; i < 16 * 784; i += kMlpFwdThreads) Ws[i] = c->params[d.w1 + (int64_t)n0 * 784 + i];
  if (threadIdx.x < 256) lut[threadIdx.x] = px01((uint8_t)threadIdx.x);
  for (int i = threadIdx.x; i < rows * 49; i += kMlpFwdThreads) {  // 784 = 49 x 16 bytes per row
    const int r = i / 49, q = i - r * 49;
    reinterpret_cast<uint4*>(xs + r * 784)[q] =
        __ldg(reinterpret_cast<const uint4*>(c->x + (int64_t)c->perm[tk.base + r] * 784) + q);
  }
  __syncthreads();
  T* h = (T*)c->buf[B_H1];
  for (int o = threadIdx.x; o < rows * 16; o += kMlpFwdThreads) {
    const int r = o >> 4, n = o & 15;
    const float* w = Ws + n * 784;
    const uint8_t* x = xs + r * 784;
    float acc = 0.f;
#pragma unroll 8
    for (int k = 0; k < 784; ++k) acc = fmaf(lut[x[k]], w[k], acc);
    stv(h + (int64_t)r * 64 + n0 + n, fmaxf(acc + c->params[d.b1 + n0 + n], 0.f));
  }
  if (threadIdx.x == 0 && c->sm_ns) atomicAdd((unsigned long long*)c->sm_ns, (unsigned long long)(globaltimer() - t_start));
}

template <typename T, int BM, int BN>
struct MlpFc1Wgrad {  // M = 64, N = 784, K = rows (fc1 bias: k_head)
  static constexpr bool A_KFAST = false, B_KFAST = false;
  const ClientRec* recs;
  MlpDims d;
  float lr;
  __device__ void setup(GemmTile& t, int local) const {
    const int nt = cdiv(784, BN);
    t.M = 64;
    t.N = 784;
    t.m0 = (local / nt) * BM;
    t.n0 = (local % nt) * BN;
    t.kb = 0;
    t.ke = t.tk.rows;
  }
  __device__ float A(const GemmTile& t, int m, int k) const {
    return ldv((const T*)t.c->buf[B_DZ1] + (int64_t)k * 64 + m);
  }
  __device__ float B(const GemmTile& t, int k, int n) const {
    const int s = t.c->perm[t.tk.base + k];
    return px01(t.c->x[(int64_t)s * 784 + n]);
  }
  __device__ void epilogue(const GemmTile& t, int mb, int nb, float acc[4][4]) const {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = mb + i, n = nb + j;
        if (m >= t.M || n >= t.N) continue;
        float* w = t.c->params + d.w1 + (int64_t)m * 784 + n;
        *w = *w - lr * acc[i][j];
      }
  }
};

// --------------------------------------------------------------------------
// Fused classifier head (K3): fc2 fwd -> softmax-CE -> dlogits -> dh (masked by
// h > 0, with the OLD W2) -> W2/b2 SGD update.  One CTA per active client.
// --------------------------------------------------------------------------
struct HeadArgs {
  const ClientRec* recs;
  int hbuf, dhbuf;  // buffer ids of h and dh (activation type T)
  int F, classes;
  int64_t w, b;     // fc2 offsets
  int64_t b_prev;   // bias of the layer producing h: b_prev -= lr * sum_r dh[r]
  float lr;
};
constexpr int kHeadThreads = 256;
template <typename T>
__global__ void __launch_bounds__(kHeadThreads) k_head(HeadArgs a, const Task* __restrict__ tasks) {
  __shared__ float dlog[64 * 64];
  __shared__ float lossr[64];
  const Task tk = tasks[blockIdx.x];
  const ClientRec* c = a.recs + tk.rec;
  const int rows = tk.rows, F = a.F, C = a.classes;
  const T* h = (const T*)c->buf[a.hbuf];
  float* W = c->params + a.w;
  float* bias = c->params + a.b;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // 1. logits
  for (int idx = warp; idx < rows * C; idx += kHeadThreads / 32) {
    const int r = idx / C, cc = idx - r * C;
    float s = 0.f;
    for (int f = lane; f < F; f += 32) s = fmaf(ldv(h + (int64_t)r * F + f), W[(int64_t)cc * F + f], s);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) dlog[r * C + cc] = s + bias[cc];
  }
  __syncthreads();
  // 2. softmax-CE per row; dlogits = (p - onehot) / rows
  if (threadIdx.x < rows) {
    const int r = threadIdx.x;
    const int label = c->y[c->perm[tk.base + r]];
    float mx = -INFINITY;
    for (int cc = 0; cc < C; ++cc) mx = fmaxf(mx, dlog[r * C + cc]);
    float s = 0.f;
    for (int cc = 0; cc < C; ++cc) s += expf(dlog[r * C + cc] - mx);
    lossr[r] = logf(s) + mx - dlog[r * C + label];
    const float inv = 1.f / (s * (float)tk.den);  // |beta|: the whole batch (micro-clients too)
    for (int cc = 0; cc < C; ++cc) {
      const float p = expf(dlog[r * C + cc] - mx);
      dlog[r * C + cc] = p * inv - (cc == label ? 1.f / (float)tk.den : 0.f);
    }
  }
  __syncthreads();
  // 3. dh = (dlogits W2) * (h > 0)   (old W2); the previous layer's bias
  //    gradient sum_r dh[r][f] is applied here (its SGD update, fused).
  T* dh = (T*)c->buf[a.dhbuf];
  float* bprev = c->params + a.b_prev;
  for (int f = threadIdx.x; f < F; f += kHeadThreads) {
    float gb = 0.f;
    for (int r = 0; r < rows; ++r) {
      float s = 0.f;
      for (int cc = 0; cc < C; ++cc) s = fmaf(dlog[r * C + cc], W[(int64_t)cc * F + f], s);
      s = ldv(h + (int64_t)r * F + f) > 0.f ? s : 0.f;
      stv(dh + (int64_t)r * F + f, s);
      gb += s;
    }
    bprev[f] -= a.lr * gb;
  }
  __syncthreads();
  // 4. W2 -= lr dlogits^T h ; b2 -= lr sum_r dlogits
  for (int idx = threadIdx.x; idx < C * F; idx += kHeadThreads) {
    const int cc = idx / F, f = idx - cc * F;
    float g = 0.f;
    for (int r = 0; r < rows; ++r) g = fmaf(dlog[r * C + cc], ldv(h + (int64_t)r * F + f), g);
    W[idx] -= a.lr * g;
  }
  if (threadIdx.x < C) {
    float g = 0.f;
    for (int r = 0; r < rows; ++r) g += dlog[r * C + threadIdx.x];
    bias[threadIdx.x] -= a.lr * g;
  }
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int r = 0; r < rows; ++r) s += lossr[r];
    c->stats[0] += s / (float)tk.den;
  }
}

// --------------------------------------------------------------------------
// CNN head, one CTA per client (F <= 512 threads, one feature each):
//  1. logits = h W2^T + b2 (warp per row, lanes over features; W2 staged in smem)
//  2. softmax-CE: dlogits = (softmax - onehot) / rows, loss
//  3. thread f: dh[:, f] = (dlogits W2[:, f]) * (h[:, f] > 0) with the OLD W2,
//     fc1 bias SGD (sum_r dh[r][f]), W2[:, f] -= lr dlogits^T h[:, f]
//  4. b2 -= lr sum_r dlogits
// Every global load of a phase is independent of the phase's stores, so they are
// issued together (the former per-row global-load loops were latency bound).
// --------------------------------------------------------------------------
// --------------------------------------------------------------------------
// Evaluation head (protea_evaluate): one CTA per group of <= 64 samples: logits
// z = h W^T + b (warp per (row, class), lanes over features), per-row CE loss and
// first-maximum prediction, summed in row order (fp64 loss) into the group's slot.
// --------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256)
    k_eval_head(const ClientRec* __restrict__ recs, const Task* __restrict__ tasks, int hbuf, int F, int C,
                int64_t w, int64_t b, double* __restrict__ loss_out, uint32_t* __restrict__ correct_out) {
  __shared__ float z[64 * 64];
  __shared__ float lossr[64];
  __shared__ int okr[64];
  const Task tk = tasks[blockIdx.x];
  const ClientRec* c = recs + tk.rec;
  const int rows = tk.rows;
  const T* h = (const T*)c->buf[hbuf];
  const float* W = c->params + w;
  const float* bias = c->params + b;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int idx = warp; idx < rows * C; idx += 8) {
    const int r = idx / C, cc = idx - r * C;
    float s = 0.f;
    for (int f = lane; f < F; f += 32) s = fmaf(ldv(h + (int64_t)r * F + f), W[(int64_t)cc * F + f], s);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) z[r * C + cc] = s + bias[cc];
  }
  __syncthreads();
  if (threadIdx.x < rows) {
    const int r = threadIdx.x, label = c->y[c->perm[tk.base + r]];
    float mx = z[r * C];
    int arg = 0;
    for (int cc = 1; cc < C; ++cc)
      if (z[r * C + cc] > mx) {
        mx = z[r * C + cc];
        arg = cc;
      }
    float s = 0.f;
    for (int cc = 0; cc < C; ++cc) s += expf(z[r * C + cc] - mx);
    lossr[r] = logf(s) + mx - z[r * C + label];
    okr[r] = arg == label;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    uint32_t k = 0;
    for (int r = 0; r < rows; ++r) {
      s += (double)lossr[r];
      k += okr[r];
    }
    loss_out[blockIdx.x] = s;
    correct_out[blockIdx.x] = k;
  }
}

constexpr int kHeadCnnThreads = 512;
inline size_t head_cnn_smem(int F, int C) { return (size_t)(C * F + 64 * C + 64 + 128) * sizeof(float); }
// + the client's activations h [64][F] staged in shared memory when that still fits (kHeadStageMax)
constexpr size_t kHeadStageMax = 220 * 1024;
inline size_t head_cnn_smem_staged(int F, int C, size_t esz) { return head_cnn_smem(F, C) + 64 * (size_t)F * esz; }
template <typename T>
__global__ void __launch_bounds__(kHeadCnnThreads)
    k_head_cnn(HeadArgs a, const Task* __restrict__ tasks, int stage_h) {
  extern __shared__ float hsm[];
  pdl_wait();
  pdl_trigger();
  const Task tk = tasks[blockIdx.x];
  const ClientRec* c = a.recs + tk.rec;
  const uint64_t t_start = threadIdx.x == 0 ? globaltimer() : 0;
  const int rows = tk.rows, F = a.F, C = a.classes;
  float* Ws = hsm;              // [C][F] old W2
  float* dlog = Ws + C * F;     // [rows][C]
  float* lossr = dlog + 64 * C; // [rows]
  int* lbl = reinterpret_cast<int*>(lossr + 64);  // [rows] labels (prefetched: perm -> y is a dependent pair)
  float* b2s = lossr + 128;     // [C] fc2 bias
  const T* __restrict__ h = (const T*)c->buf[a.hbuf];
  T* __restrict__ dh = (T*)c->buf[a.dhbuf];
  float* __restrict__ W = c->params + a.w;
  float* __restrict__ bias = c->params + a.b;
  if (threadIdx.x < rows) lbl[threadIdx.x] = c->y[c->perm[tk.base + threadIdx.x]];
  if (threadIdx.x >= 256 && threadIdx.x - 256 < C) b2s[threadIdx.x - 256] = bias[threadIdx.x - 256];
  if (stage_h) {  // h read once with 16-byte loads (every row is re-read C + 2 times below)
    T* hs = reinterpret_cast<T*>(lossr + 192);
    const int n16 = rows * F * (int)sizeof(T) / 16;
    for (int i = threadIdx.x; i < n16; i += kHeadCnnThreads)
      reinterpret_cast<uint4*>(hs)[i] = __ldg(reinterpret_cast<const uint4*>(h) + i);
    h = hs;
  }
#pragma unroll 4
  for (int i = threadIdx.x; i < C * F / 4; i += kHeadCnnThreads)  // F % 128 == 0, fc2 W 16-byte aligned
    reinterpret_cast<float4*>(Ws)[i] = reinterpret_cast<const float4*>(W)[i];
  __syncthreads();
  // 1. logits
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < rows; r += kHeadCnnThreads / 32) {
    for (int c0 = 0; c0 < C; c0 += 16) {
      float acc[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = 0.f;
#pragma unroll 4
      for (int f = lane; f < F; f += 32) {
        const float hv = ldv(h + (int64_t)r * F + f);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (c0 + j < C) acc[j] = fmaf(hv, Ws[(c0 + j) * F + f], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float v = acc[j];
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && c0 + j < C) dlog[r * C + c0 + j] = v + b2s[c0 + j];
      }
    }
  }
  __syncthreads();
  // 2. softmax cross-entropy (mean over the batch rows)
  if (threadIdx.x < rows) {
    const int r = threadIdx.x;
    const int label = lbl[r];
    float mx = -INFINITY;
    for (int cc = 0; cc < C; ++cc) mx = fmaxf(mx, dlog[r * C + cc]);
    float s = 0.f;
    for (int cc = 0; cc < C; ++cc) s += expf(dlog[r * C + cc] - mx);
    lossr[r] = logf(s) + mx - dlog[r * C + label];
    const float inv = 1.f / (s * (float)tk.den);  // |beta|: the whole batch (micro-clients too)
    for (int cc = 0; cc < C; ++cc) {
      const float p = expf(dlog[r * C + cc] - mx);
      dlog[r * C + cc] = p * inv - (cc == label ? 1.f / (float)tk.den : 0.f);
    }
  }
  __syncthreads();
  // 3. per feature: dh, fc1 bias SGD, W2 column SGD (classes in chunks of 16 register accumulators)
  const int f = threadIdx.x;
  if (f < F) {
    float gb = 0.f;
#pragma unroll 4
    for (int r = 0; r < rows; ++r) {
      const float hv = ldv(h + (int64_t)r * F + f);
      float s = 0.f;
      for (int cc = 0; cc < C; ++cc) s = fmaf(dlog[r * C + cc], Ws[cc * F + f], s);
      s = hv > 0.f ? s : 0.f;
      stv(dh + (int64_t)r * F + f, s);
      gb += s;
    }
    for (int r = rows; r < c->B; ++r) stv(dh + (int64_t)r * F + f, 0.f);  // (fc1 wgrad's TMA reads the slot's B rows)
    c->params[a.b_prev + f] -= a.lr * gb;
    for (int c0 = 0; c0 < C; c0 += 16) {
      float g[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) g[j] = 0.f;
#pragma unroll 4
      for (int r = 0; r < rows; ++r) {
        const float hv = ldv(h + (int64_t)r * F + f);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (c0 + j < C) g[j] = fmaf(dlog[r * C + c0 + j], hv, g[j]);
      }
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (c0 + j < C) W[(int64_t)(c0 + j) * F + f] = Ws[(c0 + j) * F + f] - a.lr * g[j];
    }
  }
  // 4. b2, loss statistic
  if (threadIdx.x < C) {
    float g = 0.f;
    for (int r = 0; r < rows; ++r) g += dlog[r * C + threadIdx.x];
    bias[threadIdx.x] = b2s[threadIdx.x] - a.lr * g;
  }
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int r = 0; r < rows; ++r) s += lossr[r];
    c->stats[0] += s / (float)tk.den;
    if (c->sm_ns) atomicAdd((unsigned long long*)c->sm_ns, (unsigned long long)(globaltimer() - t_start));
  }
}

}  // namespace protea
