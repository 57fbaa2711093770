// kernels_misc.cuh — admission, epoch permutation, FedAvg reduce/finalise kernels.
#pragma once
#include "device.cuh"

namespace protea {

// Admission (VCE stage (4): "another client in the round will be
// spawned"): copy the group's global weights into the client's slot and zero
// its stats.  blockIdx.y = admitted client, grid-stride over P.
__global__ void k_admit_params(const ClientRec* __restrict__ recs, const int* __restrict__ ids) {
  const ClientRec* c = recs + ids[blockIdx.y];
  const int64_t P = c->P;
  // group offsets in the global vector need not be 16-byte aligned: scalar, coalesced
  __nv_bfloat16* sh = (__nv_bfloat16*)c->buf[B_WSH];  // bf16 mode: tensor-core shadow
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const float w = c->wg[i];
    c->params[i] = w;
    if (sh) sh[i] = __float2bfloat16_rn(w);
  }
  __nv_bfloat16* w1q = (__nv_bfloat16*)c->buf[B_W1P];  // conv1 pool-quad shadow (common.h w1q_index), W1 at offset 0
  if (w1q) {
    const int C1 = c->c1, N = 4 * C1;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 288 * N; e += gridDim.x * blockDim.x) {
      const int ci = e & 7, n = (e >> 3) % N, mh = (e >> 3) / N;  // mh = (dy*3 + dx/2)*2 + dx%2
      const int dy = (mh >> 1) / 3, dx = 2 * ((mh >> 1) % 3) + (mh & 1), q = n / C1, co = n - q * C1;
      const int ky = dy - (q >> 1), kx = dx - (q & 1);
      const bool in = (unsigned)ky < 5u && (unsigned)kx < 5u && ci < 3;
      w1q[e] = __float2bfloat16_rn(in ? c->wg[co * 75 + (ky * 5 + kx) * 3 + ci] : 0.f);
    }
  }
  __nv_bfloat16* w0p = (__nv_bfloat16*)c->buf[B_R_W0P];  // ResNet conv0 [16][9][3] -> [16][9][8], W0 at offset 0
  if (w0p)
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 16 * 72; e += gridDim.x * blockDim.x) {
      const int ci = e & 7, tap = (e >> 3) % 9, co = e / 72;
      w0p[e] = __float2bfloat16_rn(ci < 3 ? c->wg[co * 27 + tap * 3 + ci] : 0.f);
    }
  if (blockIdx.x == 0 && threadIdx.x < 16) c->stats[threadIdx.x] = 0.f;
}

// Epoch permutation pi_{k,e} (reading R10): key_i = mix64(s + i*phi),
// pi = indices sorted by key (keys are distinct: mix64 is a bijection and
// s + i*phi is injective in i).  Computed as ranks: rank_i = #{j: key_j < key_i},
// pi[rank_i] = i.  blockIdx.y = admitted client, blockIdx.z = epoch.
constexpr int kPermThreads = 256, kPermChunk = 2048;
__global__ void __launch_bounds__(kPermThreads)
    k_admit_perm(const ClientRec* __restrict__ recs, const int* __restrict__ ids, uint32_t seed, uint32_t round,
                 int shuffle) {
  __shared__ uint64_t keys[kPermChunk];
  const ClientRec* c = recs + ids[blockIdx.y];
  const int e = blockIdx.z;
  if (e >= c->E) return;
  const int n = c->n;
  int32_t* perm = c->perm + (int64_t)e * n;
  const uint64_t GOLD = 0x9E3779B97F4A7C15ull;
  const uint64_t s = mix64(mix64(mix64((uint64_t)seed ^ (uint64_t)round) ^ (uint64_t)c->id) ^ (uint64_t)e);
  for (int i0 = blockIdx.x * kPermThreads; i0 < n; i0 += gridDim.x * kPermThreads) {
    const int i = i0 + threadIdx.x;
    if (!shuffle) {
      if (i < n) perm[i] = i;
      continue;
    }
    const uint64_t ki = mix64(s + (uint64_t)i * GOLD);
    int rank = 0;
    for (int j0 = 0; j0 < n; j0 += kPermChunk) {
      __syncthreads();
      for (int j = threadIdx.x; j < kPermChunk && j0 + j < n; j += kPermThreads)
        keys[j] = mix64(s + (uint64_t)(j0 + j) * GOLD);
      __syncthreads();
      const int lim = min(kPermChunk, n - j0);
      if (i < n)
        for (int j = 0; j < lim; ++j) rank += keys[j] < ki;
    }
    if (i < n) perm[rank] = i;
  }
}

// Release (P:209 stage (4) "resources get freed") + FedAvg partial:
// acc[d] += n_k * (w_k[d] - w_g[d]) in fp64, clients in the given (ascending
// id) order, so the per-element summation order is fixed.
__global__ void __launch_bounds__(256) k_release_acc(const ClientRec* __restrict__ recs, const int* __restrict__ ids,
                                                     int nrel, int64_t P, double* __restrict__ loss) {
  __shared__ const float* prm[256];  // the released clients' parameter pointers and weights, staged per chunk
  __shared__ double wn[256];
  if (loss && blockIdx.x == 0 && threadIdx.x == 0)
    for (int i = 0; i < nrel; ++i) *loss += (double)recs[ids[i]].stats[0];
  const ClientRec* c0 = recs + ids[0];
  for (int i0 = 0; i0 < nrel; i0 += 256) {  // client chunks: the per-element sum keeps the given client order
    const int nc = min(256, nrel - i0);
    __syncthreads();
    if (threadIdx.x < nc) {
      const ClientRec* c = recs + ids[i0 + threadIdx.x];
      prm[threadIdx.x] = c->params;
      wn[threadIdx.x] = (double)c->n;
    }
    __syncthreads();
    for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < P; d += (int64_t)gridDim.x * blockDim.x) {
      double a = c0->acc[d];
      const double g = (double)c0->wg[d];
      int i = 0;
      for (; i + 4 <= nc; i += 4) {  // four independent loads in flight, accumulated in order
        const float p0 = prm[i][d], p1 = prm[i + 1][d], p2 = prm[i + 2][d], p3 = prm[i + 3][d];
        a += wn[i] * ((double)p0 - g);
        a += wn[i + 1] * ((double)p1 - g);
        a += wn[i + 2] * ((double)p2 - g);
        a += wn[i + 3] * ((double)p3 - g);
      }
      for (; i < nc; ++i) a += wn[i] * ((double)prm[i][d] - g);
      c0->acc[d] = a;
    }
  }
}

// w' = w_g + acc / N  (fp64, one rounding to fp32); reading R20.
__global__ void k_finalize(const float* __restrict__ wg, const double* __restrict__ acc, double N, float* __restrict__ out,
                           int64_t P) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < P; d += (int64_t)gridDim.x * blockDim.x)
    out[d] = (float)((double)wg[d] + acc[d] / N);
}

// K7, deterministic cross-rank finalise: parts = the ranks' fp64 partials, rank r's at
// parts + r * stride; acc = ((p_0 + p_1) + p_2) + ... in rank order, then w' = w_g + acc / N (R20).
// With one part this is bitwise k_finalize (0 is not added first).
__global__ void k_finalize_ordered(const float* __restrict__ wg, const double* __restrict__ parts, int64_t stride,
                                   int nparts, double N, float* __restrict__ out, int64_t P) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < P; d += (int64_t)gridDim.x * blockDim.x) {
    double a = parts[d];
    for (int r = 1; r < nparts; ++r) a += parts[(int64_t)r * stride + d];
    out[d] = (float)((double)wg[d] + a / N);
  }
}

// protea_fedavg: out[d] = sum_k n_k p_k[d] / N, fp64 accumulation in order k.
__global__ void k_fedavg(const float* const* __restrict__ ptrs, const double* __restrict__ w, int n, double N,
                         float* __restrict__ out, int64_t dim) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < dim; d += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int k = 0; k < n; ++k) a += w[k] * (double)ptrs[k][d];
    out[d] = (float)(a / N);
  }
}

}  // namespace protea

namespace protea {

// HeteroFL-style overlapping-width aggregation for the CNN-w family (DESIGN.md reading
// R23).  Full-width (q = 4) flat index i -> flat index in the width-q sub-model (the first C1/C2/F
// channels of every hidden dimension, fc1 inputs as the first C2 channels of each of the 64 pooled
// positions), or -1 when the sub-model does not hold the element.
__device__ __forceinline__ int64_t hfl_sub_index(int64_t i, int q, int classes) {
  const int C1f = 32, C2f = 64, Ff = 512, C1 = 8 * q, C2 = 16 * q, F = 128 * q;
  int64_t so = 0;
  if (i < (int64_t)C1f * 75) return i / 75 < C1 ? i : -1;  // conv1 W [C1][5][5][3]: the first C1 rows
  i -= (int64_t)C1f * 75;
  so += (int64_t)C1 * 75;
  if (i < C1f) return i < C1 ? so + i : -1;
  i -= C1f;
  so += C1;
  if (i < (int64_t)C2f * 25 * C1f) {  // conv2 W [C2][5][5][C1]
    const int64_t co = i / (25 * C1f), r = i % (25 * C1f), tap = r / C1f, ci = r % C1f;
    return co < C2 && ci < C1 ? so + (co * 25 + tap) * C1 + ci : -1;
  }
  i -= (int64_t)C2f * 25 * C1f;
  so += (int64_t)C2 * 25 * C1;
  if (i < C2f) return i < C2 ? so + i : -1;
  i -= C2f;
  so += C2;
  if (i < (int64_t)Ff * 64 * C2f) {  // fc1 W [F][64 pooled positions][C2]
    const int64_t o = i / (64 * C2f), r = i % (64 * C2f), p = r / C2f, c = r % C2f;
    return o < F && c < C2 ? so + (o * 64 + p) * C2 + c : -1;
  }
  i -= (int64_t)Ff * 64 * C2f;
  so += (int64_t)F * 64 * C2;
  if (i < Ff) return i < F ? so + i : -1;
  i -= Ff;
  so += F;
  if (i < (int64_t)classes * Ff) {  // fc2 W [classes][F]
    const int64_t cls = i / Ff, f = i % Ff;
    return f < F ? so + cls * F + f : -1;
  }
  i -= (int64_t)classes * Ff;
  so += (int64_t)classes * F;
  return so + i;  // fc2 bias: every class
}

// out[i] = g[i] + sum_{k holds i} n_k (w_k[j_k(i)] - g[i]) / sum_{k holds i} n_k  (fp64, client order),
// or g[i] when no client holds it
__global__ void k_heterofl(const float* const* __restrict__ ptrs, const int32_t* __restrict__ wq,
                           const double* __restrict__ n, int K, const float* __restrict__ g, float* __restrict__ out,
                           int64_t P, int classes) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const double gi = (double)g[i];
    double acc = 0.0, den = 0.0;
    for (int k = 0; k < K; ++k) {
      const int64_t j = hfl_sub_index(i, wq[k], classes);
      if (j >= 0) {
        acc += n[k] * ((double)ptrs[k][j] - gi);
        den += n[k];
      }
    }
    out[i] = den > 0.0 ? (float)(gi + acc / den) : g[i];
  }
}

// the width-q sub-model of the full-width weights (what a width-q client starts from)
__global__ void k_heterofl_extract(const float* __restrict__ g, int q, int classes, float* __restrict__ sub, int64_t P) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = hfl_sub_index(i, q, classes);
    if (j >= 0) sub[j] = g[i];
  }
}

}  // namespace protea
