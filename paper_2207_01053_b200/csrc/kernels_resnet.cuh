// kernels_resnet.cuh — ResNet-8 (BASELINE.json configs[4]) grouped kernels.
//
// Model (reading R11): conv3x3 3->16, ReLU; three basic blocks
// (16, 32, 64 channels; stride 2 at blocks 2 and 3; option-A shortcut =
// subsample the block input at even pixels and append zero channels); global
// average pool; FC 64 -> classes.  Conv biases, no BatchNorm.  NHWC, weights
// [cout][ky][kx][cin].  Every 3x3 conv is an implicit GEMM on the shared SIMT
// template (k_gemm_simt) with runtime shapes:
//   fwd   M = out pixels, N = cout, K = 9 cin; epilogue bias (+ residual) + ReLU
//   dgrad M = in pixels,  N = cin,  K = 9 cout (stride-2 taps must divide);
//         epilogue (+ shortcut gradient) x ReLU mask of the stored activation
//   wgrad M = cout, N = 9 cin + 1 (bias), K = out pixels, split-K (2048 px) ->
//         partials (a region per layer) summed in split order by the step's one k_reduce_multi.
#pragma once
#include "kernels_simt.cuh"

namespace protea {

struct RConv {
  int H, W, Cin, Cout, s, Ho, Wo;  // input H x W x Cin -> output Ho x Wo x Cout, stride s, pad 1
  int64_t w, b;                    // parameter offsets
};

// forward: out = ReLU(conv(in) + b [+ res])
template <typename T, int BM, int BN>
struct RFwd {
  static constexpr bool A_KFAST = true, B_KFAST = true;
  const ClientRec* recs;
  RConv L;
  int in_buf;    // -1: the u8 input image (via the epoch permutation)
  int out_buf;
  int res_buf;   // -1 none
  int res_mode;  // 1: identity (same shape), 2: option-A shortcut from a (2Ho x 2Wo x Cres) tensor
  int Cres;
  int relu = 1;  // 0: store the raw conv output (ResNet-18: GroupNorm follows)
  __device__ void setup(GemmTile& t, int local) const {
    const int nt = cdiv(L.Cout, BN);
    t.M = t.tk.rows * L.Ho * L.Wo;
    t.N = L.Cout;
    t.m0 = (local / nt) * BM;
    t.n0 = (local % nt) * BN;
    t.kb = 0;
    t.ke = 9 * L.Cin;
  }
  __device__ float A(const GemmTile& t, int m, int k) const {
    const int hw = L.Ho * L.Wo, r = m / hw, rem = m - r * hw, yo = rem / L.Wo, xo = rem - yo * L.Wo;
    const int tap = k / L.Cin, ci = k - tap * L.Cin, ky = tap / 3, kx = tap - ky * 3;
    const int y = yo * L.s + ky - 1, x = xo * L.s + kx - 1;
    if ((unsigned)y >= (unsigned)L.H || (unsigned)x >= (unsigned)L.W) return 0.f;
    if (in_buf < 0) {
      const int smp = t.c->perm[t.tk.base + r];
      return px01(t.c->x[(int64_t)smp * L.H * L.W * L.Cin + (y * L.W + x) * L.Cin + ci]);
    }
    return ldv((const T*)t.c->buf[in_buf] + (((int64_t)r * L.H + y) * L.W + x) * L.Cin + ci);
  }
  __device__ float B(const GemmTile& t, int k, int n) const { return t.c->params[L.w + (int64_t)n * 9 * L.Cin + k]; }
  __device__ void epilogue(const GemmTile& t, int mb, int nb, float acc[4][4]) const {
    T* out = (T*)t.c->buf[out_buf];
    const int hw = L.Ho * L.Wo;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = mb + i, n = nb + j;
        if (m >= t.M || n >= t.N) continue;
        float v = acc[i][j] + t.c->params[L.b + n];
        if (res_mode == 1) {
          v += ldv((const T*)t.c->buf[res_buf] + (int64_t)m * L.Cout + n);
        } else if (res_mode == 2 && n < Cres) {
          const int r = m / hw, rem = m - r * hw, yo = rem / L.Wo, xo = rem - yo * L.Wo;
          v += ldv((const T*)t.c->buf[res_buf] + (((int64_t)r * 2 * L.Ho + 2 * yo) * 2 * L.Wo + 2 * xo) * Cres + n);
        }
        stv(out + (int64_t)m * L.Cout + n, relu ? fmaxf(v, 0.f) : v);
      }
  }
};

// dgrad: out = ([conv^T(dout)] + add) * (mask > 0)
template <typename T, int BM, int BN>
struct RDgrad {
  static constexpr bool A_KFAST = true, B_KFAST = false;
  const ClientRec* recs;
  RConv L;
  int dout_buf, out_buf, mask_buf;
  int add_buf;   // -1 none
  int add_mode;  // 1: identity (same shape as out), 2: option-A shortcut gradient from (H/2 x W/2 x Cadd)
  int Cadd;
  __device__ void setup(GemmTile& t, int local) const {
    const int nt = cdiv(L.Cin, BN);
    t.M = t.tk.rows * L.H * L.W;
    t.N = L.Cin;
    t.m0 = (local / nt) * BM;
    t.n0 = (local % nt) * BN;
    t.kb = 0;
    t.ke = 9 * L.Cout;
  }
  __device__ float A(const GemmTile& t, int m, int k) const {
    const int hw = L.H * L.W, r = m / hw, rem = m - r * hw, y = rem / L.W, x = rem - y * L.W;
    const int tap = k / L.Cout, co = k - tap * L.Cout, ky = tap / 3, kx = tap - ky * 3;
    int ty = y - ky + 1, tx = x - kx + 1;
    if (L.s == 2) {
      if ((ty | tx) & 1) return 0.f;
      ty >>= 1;
      tx >>= 1;
    }
    if ((unsigned)ty >= (unsigned)L.Ho || (unsigned)tx >= (unsigned)L.Wo) return 0.f;
    return ldv((const T*)t.c->buf[dout_buf] + (((int64_t)r * L.Ho + ty) * L.Wo + tx) * L.Cout + co);
  }
  __device__ float B(const GemmTile& t, int k, int n) const {
    const int tap = k / L.Cout, co = k - tap * L.Cout;
    return t.c->params[L.w + ((int64_t)co * 9 + tap) * L.Cin + n];
  }
  __device__ void epilogue(const GemmTile& t, int mb, int nb, float acc[4][4]) const {
    T* out = (T*)t.c->buf[out_buf];
    const T* mask = mask_buf < 0 ? nullptr : (const T*)t.c->buf[mask_buf];
    const int hw = L.H * L.W;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = mb + i, n = nb + j;
        if (m >= t.M || n >= t.N) continue;
        float v = acc[i][j];
        if (add_mode == 1) {
          v += ldv((const T*)t.c->buf[add_buf] + (int64_t)m * L.Cin + n);
        } else if (add_mode == 2) {
          const int r = m / hw, rem = m - r * hw, y = rem / L.W, x = rem - y * L.W;
          if (((y | x) & 1) == 0)
            v += ldv((const T*)t.c->buf[add_buf] +
                     (((int64_t)r * (L.H / 2) + y / 2) * (L.W / 2) + x / 2) * Cadd + n);
        }
        const int64_t o = (int64_t)m * L.Cin + n;
        stv(out + o, mask_buf < 0 || ldv(mask + o) > 0.f ? v : 0.f);  // mask_buf -1: no ReLU mask here
      }
  }
};

// wgrad split-K: partial[split][cout][9 cin + 1]
template <typename T, int BM, int BN>
struct RWgrad {
  static constexpr bool A_KFAST = false, B_KFAST = false;
  const ClientRec* recs;
  RConv L;
  int dout_buf, in_buf;  // in_buf -1: the u8 input image
  int layer;             // partial region of this layer (r8_wsp_off); -1: the start of wsp_buf
  int wsp_buf = B_R_WSP;
  __device__ void setup(GemmTile& t, int local) const {
    const int N = 9 * L.Cin + 1, nt = cdiv(N, BN), mt = cdiv(L.Cout, BM);
    t.split = local / (mt * nt);
    const int rem = local - t.split * mt * nt;
    t.M = L.Cout;
    t.N = N;
    t.m0 = (rem / nt) * BM;
    t.n0 = (rem % nt) * BN;
    if (layer >= 0) {  // ResNet-8: split = whole images [r8_split_image(s), r8_split_image(s + 1)) (common.h)
      t.kb = r8_split_image(layer, t.tk.rows, t.split) * L.Ho * L.Wo;
      t.ke = r8_split_image(layer, t.tk.rows, t.split + 1) * L.Ho * L.Wo;
    } else {  // ResNet-18: 2048-pixel splits
      t.kb = t.split * kWgradChunkPx;
      t.ke = min(t.tk.rows * L.Ho * L.Wo, t.kb + kWgradChunkPx);
    }
  }
  __device__ float A(const GemmTile& t, int m, int k) const {
    return ldv((const T*)t.c->buf[dout_buf] + (int64_t)k * L.Cout + m);
  }
  __device__ float B(const GemmTile& t, int k, int n) const {
    if (n == 9 * L.Cin) return 1.f;
    const int hw = L.Ho * L.Wo, r = k / hw, rem = k - r * hw, yo = rem / L.Wo, xo = rem - yo * L.Wo;
    const int tap = n / L.Cin, ci = n - tap * L.Cin, ky = tap / 3, kx = tap - ky * 3;
    const int y = yo * L.s + ky - 1, x = xo * L.s + kx - 1;
    if ((unsigned)y >= (unsigned)L.H || (unsigned)x >= (unsigned)L.W) return 0.f;
    if (in_buf < 0) {
      const int smp = t.c->perm[t.tk.base + r];
      return px01(t.c->x[(int64_t)smp * L.H * L.W * L.Cin + (y * L.W + x) * L.Cin + ci]);
    }
    return ldv((const T*)t.c->buf[in_buf] + (((int64_t)r * L.H + y) * L.W + x) * L.Cin + ci);
  }
  __device__ void epilogue(const GemmTile& t, int mb, int nb, float acc[4][4]) const {
    float* part = (float*)t.c->buf[wsp_buf] + (layer >= 0 ? r8_wsp_off(layer, t.c->B) : 0) +
                  (int64_t)t.split * t.M * t.N;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = mb + i, n = nb + j;
        if (m < t.M && n < t.N) part[(int64_t)m * t.N + n] = acc[i][j];
      }
  }
};

// Head: gap = mean over the 8x8 pixels of o3; logits = gap W^T + b; softmax-CE;
// dlogits; dgap = dlogits W (old W); FC SGD; ds3 = dgap/64 * (o3 > 0) -> g0.
struct RHeadArgs {
  const ClientRec* recs;
  int classes;
  int64_t w, b;
  float lr;
};
inline size_t rhead_smem(int classes) { return (size_t)(3 * 64 * 64 + 64 + classes * 64) * 4; }
template <typename T>
__global__ void __launch_bounds__(256) k_rhead(RHeadArgs a, const Task* __restrict__ tasks) {
  extern __shared__ float rh_smem[];  // rhead_smem(classes) bytes
  const Task tk = tasks[blockIdx.x];
  const ClientRec* c = a.recs + tk.rec;
  const int rows = tk.rows, C = a.classes;
  float* gap = rh_smem;           // [rows][64]
  float* dlog = gap + 64 * 64;    // [rows][C] (<= 64 x 64)
  float* lossr = dlog + 64 * 64;  // [rows]
  float* dgs = lossr + 64;        // dgap [rows][64] (shared copy for the ds3 pass)
  float* Ws = dgs + 64 * 64;      // the FC weights [C][64] (old W: logits and dgap)
  const T* o3 = (const T*)c->buf[B_R_O3];
  float* W = c->params + a.w;
  float* bias = c->params + a.b;
  for (int idx = threadIdx.x; idx < C * 64; idx += 256) Ws[idx] = W[idx];  // (offset not 16-byte aligned)
  // GAP: one (row, 16-byte channel group) per item, the 64 pixels as independent 16-byte loads, summed
  // per channel in pixel order (the same fp32 order as a scalar loop over p)
  constexpr int V = 16 / sizeof(T), G = 64 / V;
  for (int it = threadIdx.x; it < rows * G; it += 256) {
    const int r = it / G, cg = it - r * G;
    const uint4* src = reinterpret_cast<const uint4*>(o3 + (int64_t)r * 4096 + cg * V);
    float s[V];
#pragma unroll
    for (int j = 0; j < V; ++j) s[j] = 0.f;
#pragma unroll
    for (int p0 = 0; p0 < 64; p0 += 16) {
      uint4 v[16];
#pragma unroll
      for (int p = 0; p < 16; ++p) v[p] = src[(p0 + p) * G];
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        const T* e = reinterpret_cast<const T*>(&v[p]);
#pragma unroll
        for (int j = 0; j < V; ++j) s[j] += ldv(e + j);
      }
    }
#pragma unroll
    for (int j = 0; j < V; ++j) gap[r * 64 + cg * V + j] = s[j] * (1.f / 64.f);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < rows * C; idx += 256) {
    const int r = idx / C, cc = idx - r * C;
    float s = bias[cc];
    for (int f = 0; f < 64; ++f) s = fmaf(gap[r * 64 + f], Ws[cc * 64 + f], s);
    dlog[idx] = s;
  }
  __syncthreads();
  if (threadIdx.x < rows) {
    const int r = threadIdx.x, label = c->y[c->perm[tk.base + r]];
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
  // dgap = dlogits W (old W), kept in the slot's dgap buffer
  float* dgap = (float*)c->buf[B_R_DGAP];
  for (int idx = threadIdx.x; idx < rows * 64; idx += 256) {
    const int r = idx >> 6, ch = idx & 63;
    float dg = 0.f;
    for (int cc = 0; cc < C; ++cc) dg = fmaf(dlog[r * C + cc], Ws[cc * 64 + ch], dg);
    dgap[idx] = dg;
    dgs[idx] = dg;
  }
  __syncthreads();
  // ds3 = dgap / 64 * (o3 > 0)  -> g0
  T* g0 = (T*)c->buf[B_R_G0];
  // (V: elements per 16-byte vector, as above)
  const int nv = rows * 64 * 64 / V;
  for (int b0 = 0; b0 < nv; b0 += 256 * 8) {  // 8 independent 16-byte loads in flight per thread
    uint4 ov[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int iv = b0 + u * 256 + threadIdx.x;
      if (iv < nv) ov[u] = reinterpret_cast<const uint4*>(o3)[iv];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int iv = b0 + u * 256 + threadIdx.x;
      if (iv >= nv) break;
      const int idx = iv * V, r = idx >> 12, ch = idx & 63;
      const T* o = reinterpret_cast<const T*>(&ov[u]);
      uint4 gv;
      T* gq = reinterpret_cast<T*>(&gv);
#pragma unroll
      for (int j = 0; j < V; ++j) stv(gq + j, ldv(o + j) > 0.f ? dgs[r * 64 + ch + j] * (1.f / 64.f) : 0.f);
      reinterpret_cast<uint4*>(g0)[iv] = gv;
    }
  }
  for (int idx = threadIdx.x; idx < C * 64; idx += 256) {
    const int cc = idx >> 6, f = idx & 63;
    float g = 0.f;
    for (int r = 0; r < rows; ++r) g = fmaf(dlog[r * C + cc], gap[r * 64 + f], g);
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

}  // namespace protea
