// kernels_misc.cuh — admission, epoch permutation, FedAvg reduce/finalise kernels.
#pragma once
#include "device.cuh"

namespace protea {

// Admission (VCE stage (4): "another client in the round will be
// spawned"): copy the group's global weights into the client's slot and zero
// its stats.  blockIdx.y = admitted client, grid-stride over P.
// (also the micro-client broadcast after a merge: src = the merged weights, stats untouched)
__device__ __forceinline__ void load_weights(const ClientRec* c, const float* __restrict__ src, bool admit) {
  const int64_t P = c->P;
  // group offsets in the global vector need not be 16-byte aligned: scalar, coalesced
  __nv_bfloat16* sh = (__nv_bfloat16*)c->buf[B_WSH];  // bf16 mode: tensor-core shadow
  float* mw = admit ? c->mw : nullptr;                  // micro-client 0: the merge weights start as w_g
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const float w = src[i];
    if ((uint64_t)(i - c->sp_off) < (uint64_t)c->sp_len) {
      set_master_w(c, i, w);  // split planes: the hi plane is the tensor-core operand (no shadow)
    } else {
      c->params[i] = w;
      if (sh) sh[i] = __float2bfloat16_rn(w);
    }
    if (mw) mw[i] = w;
  }
  __nv_bfloat16* w1q = (__nv_bfloat16*)c->buf[B_W1P];  // conv1 pool-quad shadow (common.h w1q_index), W1 at offset 0
  if (w1q) {
    const int C1 = c->c1, N = 4 * C1;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 288 * N; e += gridDim.x * blockDim.x) {
      const int ci = e & 7, n = (e >> 3) % N, mh = (e >> 3) / N;  // mh = (dy*3 + dx/2)*2 + dx%2
      const int dy = (mh >> 1) / 3, dx = 2 * ((mh >> 1) % 3) + (mh & 1), q = n / C1, co = n - q * C1;
      const int ky = dy - (q >> 1), kx = dx - (q & 1);
      const bool in = (unsigned)ky < 5u && (unsigned)kx < 5u && ci < 3;
      w1q[e] = __float2bfloat16_rn(in ? src[co * 75 + (ky * 5 + kx) * 3 + ci] : 0.f);
    }
  }
  __nv_bfloat16* w0p = (__nv_bfloat16*)c->buf[B_R_W0P];  // ResNet conv0 [16][9][3] -> [16][9][8], W0 at offset 0
  if (w0p)
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 16 * 72; e += gridDim.x * blockDim.x) {
      const int ci = e & 7, tap = (e >> 3) % 9, co = e / 72;
      w0p[e] = __float2bfloat16_rn(ci < 3 ? src[co * 27 + tap * 3 + ci] : 0.f);
    }
  if (admit && blockIdx.x == 0 && threadIdx.x < 16) c->stats[threadIdx.x] = 0.f;
}
__global__ void k_admit_params(const ClientRec* __restrict__ recs, const int* __restrict__ ids) {
  const ClientRec* c = recs + ids[blockIdx.y];
  load_weights(c, c->wg, true);
}

// Micro-clients of one batch (common.h kMicroRows): list = [M recs][M rows], micro 0 first.  Every micro
// took its SGD step from the same weights w (= mw of micro 0) with its rows' losses divided by the WHOLE
// batch's |beta| (Task.den: the gradient tensors it stores, and rounds in bf16 mode, are the whole batch's)
// and lr * kMicroLrScale (a power of two: exact), so (w_m - w) / kMicroLrScale = -lr * (sum of micro m's
// rows' gradients) / |beta| to fp32 rounding of the SCALED step (relative eps, not ulp(w)); the merge forms,
// in fp64 and in micro order,
//   w' = w + sum_m (w_m - w) / kMicroLrScale = w - lr * (mean gradient over the whole batch),
// rounded once to fp32.  Micros without rows in this batch left w_m = w.
// Block 0 also folds the micro-batch losses (already / |beta|) into micro 0's stats[0].
__global__ void k_micro_merge(const ClientRec* __restrict__ recs, const int* __restrict__ list, int M, int R) {
  const ClientRec* c0 = recs + list[0];
  float* mw = c0->mw;
  const int64_t P = c0->P;
  const double inv = 1.0 / (double)kMicroLrScale;
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < P; d += (int64_t)gridDim.x * blockDim.x) {
    const double w = (double)mw[d];
    double a = 0.0;
    for (int m = 0; m < M; ++m)
      if (list[M + m]) a += (double)master_w(recs + list[m], d) - w;
    mw[d] = (float)(w + a * inv);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // stats[0] of micro 0 holds the client's running total (stats[1]) plus this step's micro-0 loss
    float* s0 = c0->stats;
    double step = (double)s0[0] - (double)s0[1];
    for (int m = 1; m < M; ++m) {
      float* sm = recs[list[m]].stats;
      step += (double)sm[0];
      sm[0] = 0.f;
    }
    s0[1] = (float)((double)s0[1] + step);
    s0[0] = s0[1];
  }
  (void)R;
}
// ... then every micro (blockIdx.y) reloads the merged weights (params, bf16 shadows)
__global__ void k_micro_bcast(const ClientRec* __restrict__ recs, const int* __restrict__ list) {
  const ClientRec* c = recs + list[blockIdx.y];
  load_weights(c, recs[list[0]].mw, false);
}

// Observed arena high-water marks (Table 1 "VRAM" P:140-156, get_properties P:217: "how much
// VRAM is the training making use of"; reading R2 = the peak).  A slot is filled with the poison
// byte before the client is admitted; after it is released the highest byte of the slot that differs from
// the poison bounds everything the client's kernels wrote.  regions: (byte offset in the arena, bytes,
// output index) triples, 16-byte aligned; blockIdx.y = entry of `ids` (a region index; nullptr: identity).
constexpr uint32_t kPoison4 = 0x01010101u * PROTEA_POISON;
__global__ void k_fill_poison(uint8_t* __restrict__ arena, const uint64_t* __restrict__ regions,
                              const int* __restrict__ ids) {
  const int r = ids ? ids[blockIdx.y] : (int)blockIdx.y;
  uint4* p = reinterpret_cast<uint4*>(arena + regions[3 * r]);
  const uint64_t n16 = regions[3 * r + 1] / 16;
  const uint4 v = make_uint4(kPoison4, kPoison4, kPoison4, kPoison4);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
// out[idx] = max(out[idx], 1 + offset of the highest non-poison byte of the region) (0: untouched)
__global__ void __launch_bounds__(256) k_scan_poison(const uint8_t* __restrict__ arena,
                                                     const uint64_t* __restrict__ regions, const int* __restrict__ ids,
                                                     unsigned long long* __restrict__ out) {
  const int r = ids ? ids[blockIdx.y] : (int)blockIdx.y;
  const uint4* p = reinterpret_cast<const uint4*>(arena + regions[3 * r]);
  const uint64_t n16 = regions[3 * r + 1] / 16;
  unsigned long long best = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 v = p[i];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 3; k >= 0; --k)
      if (w[k] != kPoison4) {  // little endian: the highest differing byte of word k
        const int hb = (31 - __clz(w[k] ^ kPoison4)) >> 3;
        best = max(best, (unsigned long long)(i * 16 + 4 * k + hb + 1));
        break;
      }
  }
  for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best) atomicMax(out + regions[3 * r + 2], best);
}

// Evaluate round (PAPER.md P:302 validation split, P:238 configure_evaluate / aggregate_evaluate): the
// classifier head after the training path's forward kernels.  Per row r of the task: features g (the
// stored activation row [F], or for ResNet-8 the global average over hw positions of [hw][F]), logits
// z = W g + b (fp32), loss = logsumexp(z) - z[y], correct = (first maximum of z == y).  One CTA per task,
// a warp per row; thread 0 adds the rows' losses and hits in row order to stats[0] / stats[2].
constexpr int kEvalThreads = 256;
template <typename T>
__global__ void __launch_bounds__(kEvalThreads)
    k_eval_head(const ClientRec* __restrict__ recs, const Task* __restrict__ tasks, int feat_buf, int F, int hw,
                int64_t off_w, int64_t off_b, int C) {
  __shared__ float g[kEvalThreads / 32][512];
  __shared__ float z[kEvalThreads / 32][64];
  __shared__ float loss_r[kMicroRows];
  __shared__ int ok_r[kMicroRows];
  const Task tk = tasks[blockIdx.x];
  const ClientRec* c = recs + tk.rec;
  const T* feat = (const T*)c->buf[feat_buf];
  const float* W = c->params + off_w;
  const float* bias = c->params + off_b;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < tk.rows; r += kEvalThreads / 32) {
    for (int f = lane; f < F; f += 32) {
      float a = 0.f;
      for (int p = 0; p < hw; ++p) a += ldv(feat + ((int64_t)r * hw + p) * F + f);
      g[warp][f] = hw > 1 ? a / (float)hw : a;
    }
    __syncwarp();
    for (int k = 0; k < C; ++k) {
      float a = 0.f;
      for (int f = lane; f < F; f += 32) a = fmaf(W[(int64_t)k * F + f], g[warp][f], a);
      for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0) z[warp][k] = a + bias[k];
    }
    __syncwarp();
    if (lane == 0) {
      const int y = c->y[c->perm[tk.base + r]];
      float m = z[warp][0];
      int arg = 0;
      for (int k = 1; k < C; ++k)
        if (z[warp][k] > m) {
          m = z[warp][k];
          arg = k;
        }
      float se = 0.f;
      for (int k = 0; k < C; ++k) se += expf(z[warp][k] - m);
      loss_r[r] = logf(se) + m - z[warp][y];
      ok_r[r] = arg == y;
    }
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float ls = 0.f;
    int ok = 0;
    for (int r = 0; r < tk.rows; ++r) {
      ls += loss_r[r];
      ok += ok_r[r];
    }
    c->stats[0] += ls;
    c->stats[2] += (float)ok;
  }
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
      const uint64_t si = (uint64_t)(d - c0->sp_off);  // split-plane weights (same layout for every client)
      if (si < (uint64_t)c0->sp_len) {
        const int64_t hi_i = split_hi_index(c0, (int64_t)si);
        for (int i = 0; i < nc; ++i) {
          const uint16_t* h = reinterpret_cast<const uint16_t*>(prm[i] + c0->sp_off) + hi_i;
          a += wn[i] * ((double)split_join(h[0], h[128]) - g);
        }
        c0->acc[d] = a;
        continue;
      }
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
