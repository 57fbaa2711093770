// kernels_resnet18.cuh — ResNet-18 with GroupNorm (the paper's CIFAR model, §4.1; DESIGN.md
// reading R26): the GroupNorm forward / backward, its parameter reduce + SGD, and the classifier head.  The
// 3x3 convolutions are the generic implicit GEMMs of kernels_resnet.cuh (RFwd with relu = 0: the raw conv
// output z; RDgrad without a ReLU mask; RWgrad + k_reduce_update per layer); SIMT kernels in both precisions
// (T = float: the fp32 verify mode, T = bf16: activations and gradients stored in bf16).
//
// GroupNorm (Wu & He 2018), per sample r and group g of C / kGroups channels (N = HW C / kGroups values):
//   mean, var over the group; x^ = (z - mean) rstd, rstd = 1 / sqrt(var + 1e-5); y = gamma_c x^ + beta_c
// forward kernel: y = ReLU(GN(z) [+ shortcut]) stored, (mean, rstd) kept for the backward;
// backward kernel, g = dy * (y > 0) (and, for a block's second GroupNorm, g stored as the shortcut gradient):
//   dbeta_c = sum g, dgamma_c = sum g x^ (per-sample partials, summed in sample order by k_gn_reduce),
//   dz = rstd (g gamma - mean(g gamma) - x^ mean(g gamma x^)).
// Every sum has a fixed order (per-thread strided partials combined in thread order): bitwise reproducible.
#pragma once
#include "kernels_resnet.cuh"

namespace protea {

constexpr float kGnEps = 1e-5f;
constexpr int kGnThreads = 256;

struct GnArgs {
  const ClientRec* recs;
  int layer;          // conv layer l (0..16): statistics slot
  int HW, C, Wo;      // output map (pixels, channels, width)
  int z_buf, y_buf;   // conv output (T), activation (T)
  int64_t gam, bet;   // gamma / beta offsets in params
  int res_mode;       // fwd: 0 none, 1 identity (same shape), 2 option A from a (2Ho x 2Wo x Cres) map
  int res_buf, Cres;
  int dout_buf, dz_buf, gs_buf;  // bwd: gradient in (T), gradient out (T), shortcut gradient out (T, -1 none)
};

// sum over the block of per-thread values, fixed order (warp tree, then warps in order)
__device__ __forceinline__ float gn_block_sum(float v, float* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float s = 0.f;
  for (int w = 0; w < kGnThreads / 32; ++w) s += red[w];
  return s;
}

template <typename T>
__global__ void __launch_bounds__(kGnThreads)
    k_gn_fwd(GnArgs a, const Task* __restrict__ tasks, const int* __restrict__ prefix, int ntask) {
  __shared__ float red[kGnThreads / 32];
  const int ti = find_task(prefix, ntask, blockIdx.x);
  const Task tk = tasks[ti];
  const ClientRec* c = a.recs + tk.rec;
  const int local = blockIdx.x - __ldg(prefix + ti), r = local / kGroups, g = local - r * kGroups;
  const int Cg = a.C / kGroups, N = a.HW * Cg;
  const T* z = (const T*)c->buf[a.z_buf] + (int64_t)r * a.HW * a.C + g * Cg;
  float s = 0.f;
  for (int i = threadIdx.x; i < N; i += kGnThreads) {
    const int p = i / Cg, ch = i - p * Cg;
    s += ldv(z + (int64_t)p * a.C + ch);
  }
  const float mean = gn_block_sum(s, red) / (float)N;
  float q = 0.f;
  for (int i = threadIdx.x; i < N; i += kGnThreads) {
    const int p = i / Cg, ch = i - p * Cg;
    const float d = ldv(z + (int64_t)p * a.C + ch) - mean;
    q = fmaf(d, d, q);
  }
  const float rstd = 1.f / sqrtf(gn_block_sum(q, red) / (float)N + kGnEps);
  if (threadIdx.x == 0) {
    float* st = (float*)c->buf[B_G_ST] + (((int64_t)r * kG_Layers + a.layer) * kGroups + g) * 2;
    st[0] = mean;
    st[1] = rstd;
  }
  const float* gam = c->params + a.gam;
  const float* bet = c->params + a.bet;
  T* y = (T*)c->buf[a.y_buf] + (int64_t)r * a.HW * a.C + g * Cg;
  for (int i = threadIdx.x; i < N; i += kGnThreads) {
    const int p = i / Cg, ch = i - p * Cg, cc = g * Cg + ch;
    float v = fmaf(gam[cc], (ldv(z + (int64_t)p * a.C + ch) - mean) * rstd, bet[cc]);
    if (a.res_mode == 1) {
      v += ldv((const T*)c->buf[a.res_buf] + ((int64_t)r * a.HW + p) * a.C + cc);
    } else if (a.res_mode == 2 && cc < a.Cres) {
      const int yo = p / a.Wo, xo = p - yo * a.Wo;
      v += ldv((const T*)c->buf[a.res_buf] + (((int64_t)r * 2 * (a.HW / a.Wo) + 2 * yo) * 2 * a.Wo + 2 * xo) * a.Cres + cc);
    }
    stv(y + (int64_t)p * a.C + ch, fmaxf(v, 0.f));
  }
}

template <typename T>
__global__ void __launch_bounds__(kGnThreads)
    k_gn_bwd(GnArgs a, const Task* __restrict__ tasks, const int* __restrict__ prefix, int ntask) {
  __shared__ float red[kGnThreads / 32];
  __shared__ float pg[kGnThreads], pgx[kGnThreads];  // per-thread channel partials
  __shared__ float sg[256], sgx[256];                 // per-channel sums (Cg <= 256)
  const int ti = find_task(prefix, ntask, blockIdx.x);
  const Task tk = tasks[ti];
  const ClientRec* c = a.recs + tk.rec;
  const int local = blockIdx.x - __ldg(prefix + ti), r = local / kGroups, g = local - r * kGroups;
  const int Cg = a.C / kGroups, N = a.HW * Cg;
  const int64_t base = (int64_t)r * a.HW * a.C + g * Cg;
  const T* z = (const T*)c->buf[a.z_buf] + base;
  const T* y = (const T*)c->buf[a.y_buf] + base;
  const T* dy = (const T*)c->buf[a.dout_buf] + base;
  const float* st = (const float*)c->buf[B_G_ST] + (((int64_t)r * kG_Layers + a.layer) * kGroups + g) * 2;
  const float mean = st[0], rstd = st[1];
  const float* gam = c->params + a.gam;
  // pass 1: per-channel sums of g and g x^: thread t -> channel t % Cg, pixels t / Cg, + P, ... (P = 256 / Cg
  // threads per channel; Cg in {32, 64, 128, 256}); the shortcut gradient g is stored on the way
  const int P = kGnThreads / Cg, ch0 = threadIdx.x % Cg;
  float s1 = 0.f, s2 = 0.f;
  T* gs = a.gs_buf >= 0 ? (T*)c->buf[a.gs_buf] + base : nullptr;
  for (int p = threadIdx.x / Cg; p < a.HW; p += P) {
    const int64_t o = (int64_t)p * a.C + ch0;
    const float gv = ldv(y + o) > 0.f ? ldv(dy + o) : 0.f;
    if (gs) stv(gs + o, gv);
    s1 += gv;
    s2 = fmaf(gv, (ldv(z + o) - mean) * rstd, s2);
  }
  pg[threadIdx.x] = s1;
  pgx[threadIdx.x] = s2;
  __syncthreads();
  if (threadIdx.x < Cg) {  // the P partials of channel ch: threads ch, ch + Cg, ... in order
    float a1 = 0.f, a2 = 0.f;
    for (int k = 0; k < P; ++k) {
      a1 += pg[k * Cg + threadIdx.x];
      a2 += pgx[k * Cg + threadIdx.x];
    }
    sg[threadIdx.x] = a1;
    sgx[threadIdx.x] = a2;
  }
  __syncthreads();
  // per-sample parameter-gradient partials gnp[r][0 = gamma / 1 = beta][C]
  float* gnp = (float*)c->buf[B_G_GNP] + (int64_t)r * 2 * 512;
  for (int ch = threadIdx.x; ch < Cg; ch += kGnThreads) {
    gnp[g * Cg + ch] = sgx[ch];
    gnp[512 + g * Cg + ch] = sg[ch];
  }
  // group sums of g gamma and g gamma x^ (channel order)
  float t1 = 0.f, t2 = 0.f;
  if (threadIdx.x == 0)
    for (int ch = 0; ch < Cg; ++ch) {
      t1 = fmaf(gam[g * Cg + ch], sg[ch], t1);
      t2 = fmaf(gam[g * Cg + ch], sgx[ch], t2);
    }
  if (threadIdx.x == 0) {
    red[0] = t1 / (float)N;
    red[1] = t2 / (float)N;
  }
  __syncthreads();
  const float m1 = red[0], m2 = red[1];
  T* dz = (T*)c->buf[a.dz_buf] + base;
  for (int i = threadIdx.x; i < N; i += kGnThreads) {
    const int p = i / Cg, ch = i - p * Cg;
    const int64_t o = (int64_t)p * a.C + ch;
    const float gv = ldv(y + o) > 0.f ? ldv(dy + o) : 0.f;
    const float xh = (ldv(z + o) - mean) * rstd;
    stv(dz + o, rstd * (gv * gam[g * Cg + ch] - m1 - xh * m2));
  }
}

// GroupNorm parameters of one layer: gamma -= lr sum_r gnp[r][0][c], beta -= lr sum_r gnp[r][1][c] (sample
// order).  One CTA per task.
__global__ void __launch_bounds__(256) k_gn_reduce(const ClientRec* __restrict__ recs, const Task* __restrict__ tasks,
                                                   int C, int64_t gam, int64_t bet, float lr) {
  const Task tk = tasks[blockIdx.x];
  const ClientRec* c = recs + tk.rec;
  const float* gnp = (const float*)c->buf[B_G_GNP];
  for (int ch = threadIdx.x; ch < C; ch += 256) {
    float dg = 0.f, db = 0.f;
    for (int r = 0; r < tk.rows; ++r) {
      dg += gnp[(int64_t)r * 1024 + ch];
      db += gnp[(int64_t)r * 1024 + 512 + ch];
    }
    c->params[gam + ch] -= lr * dg;
    c->params[bet + ch] -= lr * db;
  }
}

// Head: gap = mean over the 4x4 map of the last block's output [r][16][512]; logits = gap W^T + b;
// softmax-CE (mean over |beta| = Task.den); dlogits; dgap = dlogits W (old W) -> dout = dgap / 16 on every
// pixel of the map (the last GroupNorm's backward applies the ReLU mask); FC SGD.  Dynamic smem: gap
// [rows][512] + dlog [rows][C] + losses.
struct GHeadArgs {
  const ClientRec* recs;
  int classes;
  int64_t w, b;
  float lr;
  int in_buf, dout_buf;
};
inline size_t g_head_smem(int C) { return (size_t)(64 * 512 + 64 * C + 64) * sizeof(float); }
template <typename T>
__global__ void __launch_bounds__(256) k_g_head(GHeadArgs a, const Task* __restrict__ tasks) {
  extern __shared__ float hsm[];
  const Task tk = tasks[blockIdx.x];
  const ClientRec* c = a.recs + tk.rec;
  const int rows = tk.rows, C = a.classes;
  float* gap = hsm;                 // [rows][512]
  float* dlog = gap + 64 * 512;     // [rows][C]
  float* lossr = dlog + 64 * C;     // [rows]
  const T* o = (const T*)c->buf[a.in_buf];
  float* W = c->params + a.w;
  float* bias = c->params + a.b;
  for (int idx = threadIdx.x; idx < rows * 512; idx += 256) {
    const int r = idx >> 9, ch = idx & 511;
    float s = 0.f;
    for (int p = 0; p < 16; ++p) s += ldv(o + ((int64_t)r * 16 + p) * 512 + ch);
    gap[idx] = s * (1.f / 16.f);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int idx = warp; idx < rows * C; idx += 8) {
    const int r = idx / C, cc = idx - r * C;
    float s = 0.f;
    for (int f = lane; f < 512; f += 32) s = fmaf(gap[r * 512 + f], W[(int64_t)cc * 512 + f], s);
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) dlog[idx] = s + bias[cc];
  }
  __syncthreads();
  if (threadIdx.x < rows) {
    const int r = threadIdx.x, label = c->y[c->perm[tk.base + r]];
    float mx = -INFINITY;
    for (int cc = 0; cc < C; ++cc) mx = fmaxf(mx, dlog[r * C + cc]);
    float s = 0.f;
    for (int cc = 0; cc < C; ++cc) s += expf(dlog[r * C + cc] - mx);
    lossr[r] = logf(s) + mx - dlog[r * C + label];
    const float inv = 1.f / (s * (float)tk.den);
    for (int cc = 0; cc < C; ++cc) {
      const float p = expf(dlog[r * C + cc] - mx);
      dlog[r * C + cc] = p * inv - (cc == label ? 1.f / (float)tk.den : 0.f);
    }
  }
  __syncthreads();
  T* dout = (T*)c->buf[a.dout_buf];
  for (int idx = threadIdx.x; idx < rows * 512; idx += 256) {
    const int r = idx >> 9, ch = idx & 511;
    float dg = 0.f;
    for (int cc = 0; cc < C; ++cc) dg = fmaf(dlog[r * C + cc], W[(int64_t)cc * 512 + ch], dg);
    const float v = dg * (1.f / 16.f);
    for (int p = 0; p < 16; ++p) stv(dout + ((int64_t)r * 16 + p) * 512 + ch, v);
  }
  __syncthreads();  // every dgap read the old W
  for (int idx = threadIdx.x; idx < C * 512; idx += 256) {
    const int cc = idx >> 9, f = idx & 511;
    float gsum = 0.f;
    for (int r = 0; r < rows; ++r) gsum = fmaf(dlog[r * C + cc], gap[r * 512 + f], gsum);
    W[idx] -= a.lr * gsum;
  }
  if (threadIdx.x < C) {
    float gsum = 0.f;
    for (int r = 0; r < rows; ++r) gsum += dlog[r * C + threadIdx.x];
    bias[threadIdx.x] -= a.lr * gsum;
  }
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int r = 0; r < rows; ++r) s += lossr[r];
    c->stats[0] += s / (float)tk.den;
  }
}

}  // namespace protea
