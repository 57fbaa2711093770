// kernels_resnet_tc.cuh — ResNet-8 (BASELINE.json configs[4]) 3x3 convolutions on tcgen05 (bf16 mode).
//
// Same model and data layout as kernels_resnet.cuh (reading R11: NHWC bf16 activations,
// weights [cout][ky][kx][cin], pad 1, stride 1 or 2, option-A shortcut), run as implicit GEMMs on
// the generic cp.async-fed tcgen05 GEMM (k_gemm_tc, kernels_tc.cuh): every 16-byte operand chunk is
// 8 consecutive channels of one pixel (or 8 consecutive output channels of one weight row), gathered
// straight from the client's slot; out-of-image taps and K padding are zero-filled by cp.async.
// Weights come from the bf16 shadow (B_WSH), kept in step with the fp32 master by k_reduce_update.
// Layers 1-6 gather cin in {16, 32, 64} channels straight from the activations; conv0 reads the u8
// image staged as [r][32][32][8] bf16 (k_stage_r) with its weights padded to [16][9][8] (B_R_W0P).
//   fwd   M = rows*Ho*Wo out pixels, N = cout,  K = 9 cin        (A K-major, B K-major)
//         epilogue: + bias (+ identity / option-A residual), ReLU -> bf16
//   dgrad M = rows*H*W in pixels,   N = cin,   K = 9 cout       (A K-major, B MN-major)
//         epilogue: (+ shortcut gradient) x ReLU mask of the stored activation -> bf16
//   wgrad M = 9 cin + 1 (bias row), N = cout, K = 2048-pixel split (A, B MN-major)
//         epilogue: partial[split][cout][9 cin + 1] in the layer's region (summed in split order + SGD
//         by the step's one k_reduce_multi)
#pragma once
#include "kernels_resnet.cuh"
#include "kernels_tc.cuh"

namespace protea {

// ---------------------------------------------------------------------------
// Persistent cp.async-fed tcgen05 GEMM for the gathered ResNet ops: one CTA walks a
// contiguous range of the launch's 128-row tiles (the per-CTA prologue, TMEM
// allocation and launch cost of k_gemm_tc are paid once instead of per tile — a
// 32x32x16 layer has ~70k tiles per heavy iteration).  Warps 0-15 gather every
// tile's K blocks through the STAGES ring (one 16-byte cp.async per chunk),
// warp 20 issues the MMAs into one of two TMEM accumulators, warps 16-19 drain the
// other through the op's epilogue (TMEM lane quadrant = warp % 4), so gathers,
// MMAs and epilogues of consecutive tiles overlap.
// ---------------------------------------------------------------------------
constexpr int kRpProd = 512, kRpThreads = 672;  // 16 producer + 4 epilogue + 1 MMA warps
template <int BN, int STAGES>
constexpr int rp_smem_bytes() {
  return STAGES * (128 * 64 * 2 + BN * 64 * 2) + (2 * STAGES + 4) * 8 + 16 + 1024;
}
template <int BN, int STAGES, class Op>
__global__ void __launch_bounds__(kRpThreads, 1)
    k_gemm_tc_pers(const Op op, const Task* __restrict__ tasks, const int* __restrict__ prefix, int ntask) {
  constexpr int A_BYTES = 128 * 64 * 2, B_BYTES = BN * 64 * 2, STAGE = A_BYTES + B_BYTES;
  constexpr int ACC_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : 128, TMEM_COLS = 2 * ACC_COLS;
  constexpr int LAG = (STAGES - 1) < 2 ? (STAGES - 1) : 2;
  constexpr int NA = 1024 / kRpProd;                         // A chunks per producer thread per K block
  constexpr int NB = (BN * 8 + kRpProd - 1) / kRpProd;       // B chunks
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = __ldg(prefix + ntask);
  const int g0 = (int)((int64_t)blockIdx.x * total / gridDim.x);
  const int g1 = (int)((int64_t)(blockIdx.x + 1) * total / gridDim.x);
  const uint64_t t_start = threadIdx.x == 0 ? globaltimer() : 0;
  const uint32_t bar0 = tc::smem_u32(bars);
  const uint32_t full = bar0, empty = bar0 + 8 * STAGES, acc_full = bar0 + 16 * STAGES, acc_empty = acc_full + 16;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(full + 8 * s, kRpProd);
      tc::mbar_init(empty + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(acc_full + 8 * a, 1);
      tc::mbar_init(acc_empty + 8 * a, 4);
    }
    tc::mbar_fence_init();
  }
  if (warp == kRpProd / 32 + 4) tc::tmem_alloc(tc::smem_u32(tmem_slot), TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = tc::smem_u32(smem);
  TaskCursor cur;
  cur.init(prefix, ntask, g0 < total ? g0 : total - 1);
  pdl_wait();

  if (warp < kRpProd / 32) {  // ---------------- cp.async producers
    const int tid = threadIdx.x;
    int kbg = 0;
    for (int g = g0; g < g1; ++g) {
      cur.advance(prefix, g);
      TcTile t;
      t.tk = tasks[cur.ti];
      t.c = op.recs + t.tk.rec;
      op.setup(t, g - cur.lo);
      const void* any = op.any(t);
      typename Op::PA pa[NA];
      typename Op::PB pb[NB];
      int jA;  // every A chunk of this thread has the same chunk column (q = tid + 256 u)
#pragma unroll
      for (int u = 0; u < NA; ++u) {
        int i, j;
        chunk_coords<Op::A_MN, 128>(tid + kRpProd * u, i, j);
        pa[u] = op.a_pre(t, i, j);
        jA = j;
      }
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        int i = 0, j = 0;
        if (tid + kRpProd * u < BN * 8) chunk_coords<Op::B_MN, BN>(tid + kRpProd * u, i, j);
        pb[u] = op.b_pre(t, i, j);
      }
      for (int kb = 0; kb < t.nk; ++kb, ++kbg) {
        const int s = kbg % STAGES;
        if (kbg >= STAGES) tc::mbar_wait(empty + 8 * s, ((kbg / STAGES) - 1) & 1);
        const uint32_t a_base = sbase + s * STAGE, b_base = a_base + A_BYTES;
        const typename Op::KS ks = op.a_ks(t, jA, kb);  // the K block's tap / channel state, once per thread
#pragma unroll
        for (int u = 0; u < NA; ++u) tc::cp16(a_base + 16 * (tid + kRpProd * u), op.a_src(t, pa[u], ks), any);
#pragma unroll
        for (int u = 0; u < NB; ++u)
          if (tid + kRpProd * u < BN * 8) tc::cp16(b_base + 16 * (tid + kRpProd * u), op.b_src(t, pb[u], kb), any);
        tc::cp_commit();
        if (kbg >= LAG) {
          tc::cp_wait<LAG>();
          tc::fence_proxy_async();
          tc::mbar_arrive(full + 8 * ((kbg - LAG) % STAGES));
        }
      }
    }
    tc::cp_wait<0>();
    tc::fence_proxy_async();
    for (int k = (kbg - LAG > 0 ? kbg - LAG : 0); k < kbg; ++k) tc::mbar_arrive(full + 8 * (k % STAGES));
  } else if (warp < kRpProd / 32 + 4) {  // ---------------- epilogue: TMEM quadrant warp % 4
    const int row = (warp & 3) * 32 + lane;
    int it = 0;
    for (int g = g0; g < g1; ++g, ++it) {
      cur.advance(prefix, g);
      TcTile t;
      t.tk = tasks[cur.ti];
      t.c = op.recs + t.tk.rec;
      op.setup(t, g - cur.lo);
      const int a = it & 1;
      tc::mbar_wait(acc_full + 8 * a, (it >> 1) & 1);
      tc::fence_after();
      for (int c0 = 0; c0 < t.n_mma; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(a * ACC_COLS + c0), v);
        op.epilogue(t, row, c0, v);
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(acc_empty + 8 * a);
    }
  } else {  // ---------------- MMA issuer (last warp, elected lane issues)
    const uint64_t da0 = cp_desc<Op::A_MN, 128>(sbase, 0), dak = cp_desc<Op::A_MN, 128>(sbase, 1) - da0;
    const uint64_t db0 = cp_desc<Op::B_MN, BN>(sbase + A_BYTES, 0),
                   dbk = cp_desc<Op::B_MN, BN>(sbase + A_BYTES, 1) - db0;
    int kbg = 0, it = 0;
    for (int g = g0; g < g1; ++g, ++it) {
      cur.advance(prefix, g);
      TcTile t;
      t.tk = tasks[cur.ti];
      t.c = op.recs + t.tk.rec;
      op.setup(t, g - cur.lo);
      const uint32_t idesc = tc::idesc_bf16(128, t.n_mma, Op::A_MN, Op::B_MN);
      const int a = it & 1;
      if (it >= 2) tc::mbar_wait(acc_empty + 8 * a, ((it >> 1) - 1) & 1);
      tc::fence_after();
      for (int kb = 0; kb < t.nk; ++kb, ++kbg) {
        const int s = kbg % STAGES;
        tc::mbar_wait(full + 8 * s, (kbg / STAGES) & 1);
        tc::fence_after();
        const uint64_t so = (uint64_t)(s * (STAGE >> 4));
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          tc::mma_bf16_w(tmem + (uint32_t)(a * ACC_COLS), da0 + so + ks * dak, db0 + so + ks * dbk, idesc,
                         (kb | ks) != 0);
        tc::commit_w(empty + 8 * s);
      }
      tc::commit_w(acc_full + 8 * a);
    }
    __syncwarp();
  }
  pdl_trigger();
  tc::fence_before();
  __syncthreads();
  if (warp == kRpProd / 32 + 4) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, TMEM_COLS);
  }
  if (threadIdx.x == 0 && g1 > g0) {  // K9: split this CTA's duration over its clients by tile count
    const uint64_t dt = globaltimer() - t_start;
    int ti = find_task(prefix, ntask, g0), lo = g0;
    while (lo < g1) {
      const int hi = min(g1, __ldg(prefix + ti + 1));
      const ClientRec* c = op.recs + tasks[ti].rec;
      if (c->sm_ns) atomicAdd((unsigned long long*)c->sm_ns, (unsigned long long)(dt * (hi - lo) / (g1 - g0)));
      lo = hi;
      ++ti;
    }
  }
}

struct RTcConv {  // RConv + log2 of the channel counts and of the (power-of-two) spatial sizes
  int H, W, Cin, Cout, s, Ho, Wo, lci, lco;
  int lw, lhw, lwo, lhwo;  // log2 W, log2 H*W, log2 Wo, log2 Ho*Wo
  int64_t w, b;
};

struct RTcFwd {
  static constexpr bool A_MN = false, B_MN = false;
  struct PA { const bf16* p; int y0, x0; };  // input pixel (r, y0, x0) of the row (y0 = -4096: beyond M)
  struct KS { int off, ky, kx, ok; };          // tap (ky, kx) / channel of the K block's chunk column
  struct PB { const bf16* p; int j; };
  const ClientRec* recs;
  RTcConv L;
  int in_buf, out_buf, res_buf, res_mode, Cres;  // res_mode 1: identity, 2: option-A (2Ho x 2Wo x Cres)
  int wbuf;                                      // weights [cout][9][cin] bf16: B_WSH at L.w, or B_R_W0P (conv0)
  __device__ void setup(TcTile& t, int local) const {
    t.m0 = local * 128;
    t.n0 = 0;
    t.nk = (9 * L.Cin + 63) / 64;
    t.n_mma = L.Cout;
  }
  __device__ const void* any(const TcTile& t) const { return t.c->params; }
  __device__ PA a_pre(const TcTile& t, int i, int j) const {
    const int m = t.m0 + i, hw = L.Ho * L.Wo;
    if (m >= t.tk.rows * hw) return PA{nullptr, -4096, -4096};
    const int r = m >> L.lhwo, rem = m & (hw - 1), y0 = (rem >> L.lwo) * L.s - 1, x0 = (rem & (L.Wo - 1)) * L.s - 1;
    return PA{(const bf16*)t.c->buf[in_buf] + (((int64_t)r * L.H + y0) * L.W + x0) * L.Cin, y0, x0};
  }
  __device__ KS a_ks(const TcTile& t, int j, int kb) const {
    const int k = kb * 64 + 8 * j, tap = k >> L.lci, ky = tap / 3, kx = tap - 3 * ky;
    return KS{(ky * L.W + kx) * L.Cin + (k & (L.Cin - 1)), ky, kx, k < 9 * L.Cin};
  }
  __device__ const void* a_src(const TcTile& t, const PA& s, const KS& k) const {
    if (!k.ok || (unsigned)(s.y0 + k.ky) >= (unsigned)L.H || (unsigned)(s.x0 + k.kx) >= (unsigned)L.W) return nullptr;
    return s.p + k.off;
  }
  __device__ PB b_pre(const TcTile& t, int i, int j) const {
    const bf16* w = (const bf16*)t.c->buf[wbuf] + (wbuf == B_WSH ? L.w : 0);
    return PB{i < L.Cout ? w + (int64_t)i * 9 * L.Cin + 8 * j : nullptr, j};
  }
  __device__ const void* b_src(const TcTile& t, const PB& s, int kb) const {
    return s.p && kb * 64 + 8 * s.j < 9 * L.Cin ? s.p + kb * 64 : nullptr;
  }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
    const int m = t.m0 + row, hw = L.Ho * L.Wo;
    if (m >= t.tk.rows * hw) return;
    const float* bias = t.c->params + L.b + c0;
    float o[16], q[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) o[j] = v[j] + bias[j];
    if (res_mode == 1) {
      ld_bf16<16>((const bf16*)t.c->buf[res_buf] + (int64_t)m * L.Cout + c0, q);
#pragma unroll
      for (int j = 0; j < 16; ++j) o[j] += q[j];
    } else if (res_mode == 2 && c0 < Cres) {
      const int r = m >> L.lhwo, rem = m & (hw - 1), yo = rem >> L.lwo, xo = rem & (L.Wo - 1);
      ld_bf16<16>((const bf16*)t.c->buf[res_buf] + (((int64_t)r * 2 * L.Ho + 2 * yo) * 2 * L.Wo + 2 * xo) * Cres + c0, q);
#pragma unroll
      for (int j = 0; j < 16; ++j) o[j] += q[j];
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) o[j] = fmaxf(o[j], 0.f);
    st_bf16<16>((bf16*)t.c->buf[out_buf] + (int64_t)m * L.Cout + c0, o);
  }
};

struct RTcDgrad {
  static constexpr bool A_MN = false, B_MN = true;
  struct PA { const bf16* p; int y, x; };  // dout of image r, and the input pixel (y, x) of the row
  struct KS { int ky, kx, co, ok; };
  struct PB { int i, n0; };               // k row i of the block, 8 input channels from n0
  const ClientRec* recs;
  RTcConv L;
  int dout_buf, out_buf, mask_buf, add_buf, add_mode, Cadd;
  __device__ void setup(TcTile& t, int local) const {
    t.m0 = local * 128;
    t.n0 = 0;
    t.nk = (9 * L.Cout + 63) / 64;
    t.n_mma = L.Cin;
  }
  __device__ const void* any(const TcTile& t) const { return t.c->params; }
  __device__ PA a_pre(const TcTile& t, int i, int j) const {
    const int m = t.m0 + i, hw = L.H * L.W;
    if (m >= t.tk.rows * hw) return PA{nullptr, -4096, -4096};
    const int r = m >> L.lhw, rem = m & (hw - 1);
    return PA{(const bf16*)t.c->buf[dout_buf] + (int64_t)r * L.Ho * L.Wo * L.Cout, rem >> L.lw, rem & (L.W - 1)};
  }
  __device__ KS a_ks(const TcTile& t, int j, int kb) const {
    const int k = kb * 64 + 8 * j, tap = k >> L.lco, ky = tap / 3;
    return KS{ky, tap - 3 * ky, k & (L.Cout - 1), k < 9 * L.Cout};
  }
  __device__ const void* a_src(const TcTile& t, const PA& s, const KS& k) const {
    int ty = s.y - k.ky + 1, tx = s.x - k.kx + 1;
    if (!k.ok) return nullptr;
    if (L.s == 2) {
      if ((ty | tx) & 1) return nullptr;
      ty >>= 1;
      tx >>= 1;
    }
    if ((unsigned)ty >= (unsigned)L.Ho || (unsigned)tx >= (unsigned)L.Wo) return nullptr;
    return s.p + (ty * L.Wo + tx) * L.Cout + k.co;
  }
  __device__ PB b_pre(const TcTile& t, int i, int j) const { return PB{i, 8 * j}; }
  __device__ const void* b_src(const TcTile& t, const PB& s, int kb) const {
    const int k = kb * 64 + s.i;
    if (k >= 9 * L.Cout || s.n0 >= L.Cin) return nullptr;
    const int tap = k >> L.lco, co = k & (L.Cout - 1);
    return (const bf16*)t.c->buf[B_WSH] + L.w + ((int64_t)co * 9 + tap) * L.Cin + s.n0;
  }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
    const int m = t.m0 + row, hw = L.H * L.W;
    if (m >= t.tk.rows * hw) return;
    const int64_t o = (int64_t)m * L.Cin + c0;
    float a[16], q[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = v[j];
    if (add_mode == 1) {
      ld_bf16<16>((const bf16*)t.c->buf[add_buf] + o, q);
#pragma unroll
      for (int j = 0; j < 16; ++j) a[j] += q[j];
    } else if (add_mode == 2) {
      const int r = m >> L.lhw, rem = m & (hw - 1), y = rem >> L.lw, x = rem & (L.W - 1);
      if (((y | x) & 1) == 0) {
        ld_bf16<16>((const bf16*)t.c->buf[add_buf] + (((int64_t)r * (L.H / 2) + y / 2) * (L.W / 2) + x / 2) * Cadd + c0, q);
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] += q[j];
      }
    }
    ld_bf16<16>((const bf16*)t.c->buf[mask_buf] + o, q);
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = q[j] > 0.f ? a[j] : 0.f;
    st_bf16<16>((bf16*)t.c->buf[out_buf] + o, a);
  }
};

struct RTcWgrad {
  static constexpr bool A_MN = true, B_MN = true;
  struct PA { int i, dy, dx, ci, kind; };  // kind 0: gather, 1: bias ones row, 2: zero
  struct KS { int p0; };                   // first pixel of the K block
  struct PB { int i, n0; };
  const ClientRec* recs;
  RTcConv L;
  int dout_buf, in_buf;
  int cin_real;  // channels of the weight layout (conv0: 3 real of the 8 staged; else Cin)
  int layer;     // partial region of this layer (r8_wsp_off)
  __device__ int mtiles() const { return (9 * L.Cin + 1 + 127) / 128; }
  __device__ int p0(const TcTile& t) const { return r8_split_image(layer, t.tk.rows, t.n0) * L.Ho * L.Wo; }  // (common.h)
  __device__ int p1(const TcTile& t) const { return r8_split_image(layer, t.tk.rows, t.n0 + 1) * L.Ho * L.Wo; }
  __device__ void setup(TcTile& t, int local) const {
    const int mt = mtiles(), split = local / mt;
    t.m0 = (local - split * mt) * 128;
    t.n0 = split;  // the split index (K = this split's pixels [p0, p1))
    t.nk = (p1(t) - p0(t) + 63) / 64;
    t.n_mma = L.Cout;
  }
  __device__ const void* any(const TcTile& t) const { return t.c->params; }
  __device__ PA a_pre(const TcTile& t, int i, int j) const {
    const int mg = t.m0 + 8 * j, Kw = 9 * L.Cin;
    if (mg == Kw) return PA{i, 0, 0, 0, 1};
    if (mg > Kw) return PA{i, 0, 0, 0, 2};
    const int tap = mg >> L.lci, ky = tap / 3, kx = tap - 3 * ky;
    return PA{i, ky - 1, kx - 1, mg & (L.Cin - 1), 0};
  }
  __device__ KS a_ks(const TcTile& t, int j, int kb) const { return KS{p0(t) + kb * 64}; }
  __device__ const void* a_src(const TcTile& t, const PA& s, const KS& k) const {
    if (s.kind) return s.kind == 1 ? (const void*)kOneChunk : nullptr;
    const int hw = L.Ho * L.Wo, p = k.p0 + s.i;
    if (p >= p1(t)) return nullptr;
    const int r = p >> L.lhwo, rem = p & (hw - 1), yo = rem >> L.lwo, xo = rem & (L.Wo - 1);
    const int y = yo * L.s + s.dy, x = xo * L.s + s.dx;
    if ((unsigned)y >= (unsigned)L.H || (unsigned)x >= (unsigned)L.W) return nullptr;
    return (const bf16*)t.c->buf[in_buf] + (((int64_t)r * L.H + y) * L.W + x) * L.Cin + s.ci;
  }
  __device__ PB b_pre(const TcTile& t, int i, int j) const { return PB{i, 8 * j}; }
  __device__ const void* b_src(const TcTile& t, const PB& s, int kb) const {
    const int p = p0(t) + kb * 64 + s.i;
    if (p >= p1(t) || s.n0 >= L.Cout) return nullptr;
    return (const bf16*)t.c->buf[dout_buf] + (int64_t)p * L.Cout + s.n0;
  }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
    const int m = t.m0 + row, N = 9 * cin_real + 1;  // partial row = the weight layout's K + bias
    if (m > 9 * L.Cin) return;
    const int ci = m & (L.Cin - 1), n = m == 9 * L.Cin ? 9 * cin_real : (m >> L.lci) * cin_real + ci;
    if (m < 9 * L.Cin && ci >= cin_real) return;  // padded input channels
    float* part = (float*)t.c->buf[B_R_WSP] + r8_wsp_off(layer, t.c->B) + ((int64_t)t.n0 * L.Cout + c0) * N + n;
#pragma unroll
    for (int j = 0; j < 16; ++j) part[(int64_t)j * N] = v[j];
  }
};

// conv0 input staged for the tensor cores: xs[r][32][32][8] bf16 = px01(x) in channels 0-2, 0 in 3-7
// (written into a gradient buffer that is free at that point of the step).  blockIdx.x = task.
__global__ void __launch_bounds__(256) k_stage_r(const ClientRec* __restrict__ recs, const Task* __restrict__ tasks,
                                                 int out_buf) {
  const Task tk = tasks[blockIdx.x];
  const ClientRec* c = recs + tk.rec;
  uint4* out = (uint4*)c->buf[out_buf];
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < tk.rows * 1024; e += gridDim.y * blockDim.x) {
    const int r = e >> 10, p = e & 1023;
    const uint8_t* px = c->x + (int64_t)c->perm[tk.base + r] * 3072 + p * 3;
    const __nv_bfloat162 a = __floats2bfloat162_rn(px01(px[0]), px01(px[1]));
    const __nv_bfloat162 b = __floats2bfloat162_rn(px01(px[2]), 0.f);
    out[e] = make_uint4(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b), 0u, 0u);
  }
}

}  // namespace protea
