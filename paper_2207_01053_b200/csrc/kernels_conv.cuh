// kernels_conv.cuh — persistent "halo" implicit-GEMM 5x5 convolutions on tcgen05 (bf16 mode).
//
// conv1 fwd (M = output pixels, N = C1, K = 25 taps x 3 (padded 8) ch), conv2 fwd
// (N = C2, K = 25 x C1) and conv2 dgrad (M = a1 pixels, N = C1, K = 25 x C2)
// re-read every input element once per tap when the im2col operand is gathered
// per K block.  Here:
//  * a PERSISTENT CTA (one per SM) walks a contiguous range of the iteration's
//    128-pixel tiles (8 image rows x 16 columns), client after client;
//  * the weight operand of the current client (all 25 taps) is loaded once by
//    TMA and stays resident in shared memory until the range moves to the
//    next client (b_full / b_empty barriers);
//  * per tile (and per 32-channel group of the input) the TMA loads the input
//    halo ONCE as 5 x-shifted copies (out-of-bounds rows / columns are the
//    TMA's zero fill = the conv padding); the A operand of tap (ky, kx) is then
//    only a UMMA descriptor into copy kx starting at row ky;
//  * the halo is double-buffered and the fp32 accumulator double-buffered in
//    TMEM, so TMA, tcgen05.mma and the epilogue of the previous tile overlap.
// Warp roles: warps 0-7 epilogue (tcgen05.ld + fused layer epilogue), warp 8
// lane 0 TMA producer, warp 9 lane 0 MMA issuer.
#pragma once
#include "kernels_tc.cuh"

namespace protea {

#ifndef PROTEA_DBG
#define PROTEA_DBG 0
#endif
__device__ unsigned long long g_dbg[64];  // PROTEA_DBG cycle counters (protea_debug_counters)
#define DBG_T0(v) const long long v = PROTEA_DBG ? clock64() : 0
#define DBG_ADD(i, v) \
  if (PROTEA_DBG && (threadIdx.x & 31) == 0) atomicAdd(&g_dbg[i], (unsigned long long)(clock64() - (v)))


constexpr int kConvThreads = 320;
// dgrad epilogue operands: loaded one tile ahead (true) or at the start of the tile's epilogue,
// before its accumulator wait (false).  Measured on B200: the one-tile-ahead variant was slower.
constexpr bool kCrossTilePrefetch = false;
template <class Op>
struct xprefetch {  // k_conv_persistent loads tile g + 1's epilogue operands (Op::prefetch) before tile g's epilogue
  template <class U>
  static constexpr bool f(decltype(U::XPF)*) { return U::XPF; }
  template <class U>
  static constexpr bool f(...) { return kCrossTilePrefetch; }
  static constexpr bool value = f<Op>(nullptr);
};

// ---------------------------------------------------------------------------
// conv2 fwd / dgrad
// ---------------------------------------------------------------------------
template <int CIN>  // channels of the gathered input (per 32-channel halo group)
struct HaloGeom {
  // CIN >= 32: one TMA box (32 ch, 16 px, 12 rows) per x-shift, 64-byte swizzled (64 B pixel rows);
  // otherwise 8-channel boxes with 16-byte pixel rows (no swizzle).
  static constexpr bool SW64 = CIN >= 32;
  static constexpr int NCC = CIN < 32 ? CIN / 8 : 4;  // 8-channel chunks per halo group
  static constexpr int GROUPS = CIN / (8 * NCC);       // halo groups per tile
  static constexpr int ROWS = 12;                      // 8 output rows + 4 halo rows
  static constexpr int COPY = ROWS * 16 * 16;          // bytes of one (kx, 8-channel chunk) copy
  static constexpr int BYTES = 5 * NCC * COPY;         // one halo buffer
};

// Fwd: input a1 (C1 channels), weights K-major [kchunk][C2][8]; epilogue bias + ReLU + 2x2 pool -> a2, i2.
// Dgrad: input dz2 (C2 channels, flipped taps), weights MN-major [tap][C1/8][C2][8]; epilogue ReLU mask
// + pool-1 backward scatter -> dz1 (width 1: in the pool-quad layout of k_conv1_wgrad_q).
template <int WQ, bool DGRAD>
struct HaloConv2 {
  typedef CnnW<WQ> W;
  static constexpr int CIN = DGRAD ? W::C2 : W::C1;   // gathered input channels
  static constexpr int NOUT = DGRAD ? W::C1 : W::C2;  // valid output channels
  static constexpr int N = NOUT < 16 ? 16 : NOUT;     // MMA N
  static constexpr bool B_MN = DGRAD;
  typedef HaloGeom<CIN> G;
  static constexpr int GROUPS = G::GROUPS;
  static constexpr int HBYTES = G::BYTES;
  static constexpr int B_BYTES = 25 * CIN * N * 2;    // resident weights (K x N bf16)
  static constexpr int TMEM_COLS = 2 * N <= 32 ? 32 : 2 * N <= 64 ? 64 : 2 * N <= 128 ? 128 : 256;
  static constexpr int SMEM = B_BYTES + 2 * HBYTES + 256 + 1024;  // + realignment slack
  static constexpr int HSTRIDE = HBYTES, BSTRIDE = B_BYTES;        // buffer strides (= the TMA bytes)
  static constexpr int TILES_PER_IMAGE = 2;
  static constexpr int DBG = DGRAD ? 32 : 16;
  const ClientRec* recs;
  CnnDims d;

  __device__ void load_b(const TcTile& t, uint32_t sb, uint32_t bar) const {
    if (!DGRAD) {  // [kchunk][C2][8]: box (8, C2) per 8-wide K chunk
      for (int kc = 0; kc < 25 * W::C1 / 8; ++kc) tc::tma_load_2d(sb + kc * N * 16, tmap_of(t, TM_W2F), bar, 8 * kc, 0);
    } else {  // [tap][C1/8 (padded to N/8)][C2][8]: box (8 ci, 1 tap, C2 co)
      for (int tap = 0; tap < 25; ++tap)
        for (int nc = 0; nc < N / 8; ++nc)
          tc::tma_load_3d(sb + (tap * (N / 8) + nc) * W::C2 * 16, tmap_of(t, TM_W2D), bar, 8 * nc, tap, 0);
    }
  }
  __device__ void load_halo(const TcTile& t, int tile, int grp, uint32_t base, uint32_t bar) const {
    const void* tin = tmap_of(t, DGRAD ? TM_DZ2H : TM_A1H);
    const int r = tile >> 1, y0 = (tile & 1) * 8;
    if constexpr (G::SW64) {
      for (int kx = 0; kx < 5; ++kx)  // copy kx = [12 rows][16 px][32 ch], 64 B swizzled
        tc::tma_load_4d(base + kx * 4 * G::COPY, tin, bar, 32 * grp, DGRAD ? 2 - kx : kx - 2, y0 - 2, r);
    } else {
      for (int kx = 0; kx < 5; ++kx)
        for (int cc = 0; cc < G::NCC; ++cc)
          tc::tma_load_4d(base + (kx * G::NCC + cc) * G::COPY, tin, bar, 8 * (grp * G::NCC + cc),
                          DGRAD ? 2 - kx : kx - 2, y0 - 2, r);
    }
  }
  __device__ void mma_stage(uint32_t hb, uint32_t sb, uint32_t dt, int grp, uint32_t idesc, int = 0) const {
    const uint64_t a0 = G::SW64 ? tc::sdesc_sw64(hb, 16, 512) : tc::sdesc(hb, G::COPY, 128);
    const uint64_t b0 = !DGRAD ? tc::sdesc(sb + grp * G::NCC * N * 16, N * 16, 128)  // K chunk (tap, grp*NCC + 2cp)
                               : tc::sdesc(sb + grp * G::NCC * 128, 128, W::C2 * 16);  // k rows = co of tap
#pragma unroll
    for (int ky = 0; ky < 5; ++ky)
#pragma unroll
      for (int kx = 0; kx < 5; ++kx) {
        const int tap = ky * 5 + kx, row0 = DGRAD ? 4 - ky : ky;
#pragma unroll
        for (int cp = 0; cp < G::NCC / 2; ++cp) {
          const uint32_t ao = G::SW64 ? kx * 4 * G::COPY + row0 * 1024 + 32 * cp
                                      : (kx * G::NCC + 2 * cp) * G::COPY + row0 * 256;
          const uint32_t bo = !DGRAD ? (tap * (W::C1 / 8) + 2 * cp) * N * 16 : tap * (N / 8) * W::C2 * 16 + cp * 256;
          tc::mma_bf16_w(dt, tc::dadd(a0, ao), tc::dadd(b0, bo), idesc, (grp | tap | cp) != 0);
        }
      }
  }
  // Epilogue of one tile: warps w, w+4 share TMEM lanes; column chunks c0 = 16 g + 32 j.
  static constexpr int NCH = (N + 31) / 32;
  static constexpr int NV = NOUT < 16 ? NOUT : 16;
  struct EpiState {  // per-client values cached across the tiles of a client (the bias)
    const ClientRec* c = nullptr;
    float bias[NCH][16];
  };
  // dgrad: the pool-1 operands (a1 > 0 mask, argmax) of the NEXT tile are loaded into registers
  // while the current tile is processed (the epilogue, not the MMA, is the critical path).
  struct Pre {
    uint4 a[NCH][2];
    uint4 i[NCH];
  };
  __device__ void prefetch(const TcTile& t, int tile, int warp, int lane, Pre& p) const {
    if constexpr (DGRAD) {
      const int g = warp >> 2, m = tile * 128 + (warp & 3) * 32 + lane;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const int c0 = g * 16 + 32 * j;
        if (c0 >= N) continue;
        const int64_t o = (int64_t)m * W::C1 + c0;
        const uint4* a = reinterpret_cast<const uint4*>((const bf16*)t.c->buf[B_A1] + o);
        p.a[j][0] = a[0];
        if (NV == 16) p.a[j][1] = a[1];
        if (NV == 16)
          p.i[j] = *reinterpret_cast<const uint4*>((const uint8_t*)t.c->buf[B_I1] + o);
        else {
          const uint2 u = *reinterpret_cast<const uint2*>((const uint8_t*)t.c->buf[B_I1] + o);
          p.i[j] = make_uint4(u.x, u.y, 0, 0);
        }
      }
    }
  }
  __device__ void epilogue(const TcTile& t, int tile, uint32_t tacc, uint32_t full_bar, uint32_t parity, int warp,
                           int lane, EpiState& st, const Pre& pre) const {
    const int g = warp >> 2, row = (warp & 3) * 32 + lane;
    const int m = tile * 128 + row, r = m >> 8, y = (m >> 4) & 15, x = m & 15;
    float a1v[NCH][NV];
    int argv[NCH][NV];
    if (!DGRAD && st.c != t.c) {
      st.c = t.c;
#pragma unroll
      for (int j = 0; j < NCH; ++j)
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int n = g * 16 + 32 * j + q;
          st.bias[j][q] = (q < NV && n < NOUT) ? t.c->params[d.b2 + n] : 0.f;
        }
    }
    if (DGRAD) {
      Pre now;
      if constexpr (!kCrossTilePrefetch) prefetch(t, tile, warp, lane, now);  // before waiting on the MMA
      const Pre& p = kCrossTilePrefetch ? pre : now;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        ld_bf16<NV>(reinterpret_cast<const bf16*>(&p.a[j][0]), a1v[j]);
        ld_u8<NV>(reinterpret_cast<const uint8_t*>(&p.i[j]), argv[j]);
      }
    }
    tc::mbar_wait(full_bar, parity);
    tc::fence_after();
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c0 = g * 16 + 32 * j;
      if (c0 >= N) continue;
      float v[16];
      tc::tmem_ld16(tacc + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0, v);
      if (DGRAD) {  // pool-1 backward: dz1 = scatter(v * (a1 > 0)) to the argmax of each 2x2 window
        bf16* dz1 = (bf16*)t.c->buf[B_DZC1];
        float out[NV];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int e = 0; e < NV; ++e) out[e] = (argv[j][e] == q && a1v[j][e] > 0.f) ? v[e] : 0.f;
          if constexpr (WQ == 4) {  // pool-quad layout g1[r][py][px][q][C1] (k_conv1_wgrad_q)
            st_bf16<NV>(dz1 + (((int64_t)r * 256 + y * 16 + x) * 4 + q) * W::C1 + c0, out);
          } else {  // full-resolution dz1[r][Y][X][C1] (TcConv1Wgrad)
            const int Y = 2 * y + (q >> 1), X = 2 * x + (q & 1);
            st_bf16<NV>(dz1 + ((int64_t)r * 1024 + Y * 32 + X) * W::C1 + c0, out);
          }
        }
      } else {  // bias + ReLU + 2x2 max-pool (first max) over lanes (l, l+1, l+16, l+17)
        const int base = lane & 14;
        float val[16], best[16];
        int arg[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) val[e] = e < NV ? fmaxf(v[e] + st.bias[j][e], 0.f) : 0.f;
        pool_lanes(val, base, base + 1, base + 16, base + 17, best, arg);
        if (lane < 16 && (lane & 1) == 0) {
          const int64_t o = ((int64_t)r * 64 + (y >> 1) * 8 + (x >> 1)) * W::C2 + c0;
          st_bf16<NV>((bf16*)t.c->buf[B_A2] + o, best);
          st_u8<NV>((uint8_t*)t.c->buf[B_I2] + o, arg);
        }
      }
    }
  }
};

// ---------------------------------------------------------------------------
// conv2 fwd / dgrad, width 1 (C1 = 32, C2 = 64), single-halo form.  Tile = 16 output
// rows x 8 columns (one image half), M row m = y * 8 + x.  Per 32-channel group ONE TMA
// box brings the input halo [20 rows][12 px][32 ch] (64-byte swizzle) and every tap's A
// operand is a descriptor into it, shifted by whole 64-byte pixel rows (the swizzle
// follows absolute addresses: tools/swz_test.cu): K-major, 8-row core groups = 8 pixels
// of one halo row (SBO = 768 B = one halo row), K step 16 channels = +32 B.  The
// weights are loaded by a few wide boxes: fwd K-major 128-byte swizzle [13][64 co][64 k]
// (8 KB per 64-wide K block), dgrad MN-major 64-byte swizzle [25 taps][64 co][32 ci].
// Pool partners (y,x),(y,x+1),(y+1,x),(y+1,x+1) are lanes l, l+1, l+8, l+9.
// ---------------------------------------------------------------------------
template <bool DGRAD>
struct HaloConv2Q {
  typedef CnnW<4> W;
  static constexpr int CIN = DGRAD ? 64 : 32;
  static constexpr int NOUT = DGRAD ? 32 : 64, N = NOUT;
  static constexpr bool B_MN = DGRAD;
  static constexpr int GROUPS = CIN / 32;
  static constexpr int HALO = 20 * 12 * 64;           // one 32-channel group
  static constexpr int HBYTES = HALO;                 // one pipeline stage = one group's halo
  static constexpr int B_BYTES = DGRAD ? 25 * 4096 : 13 * 8192;
  static constexpr int TMEM_COLS = 2 * N <= 64 ? 64 : 128;
  static constexpr int SMEM = B_BYTES + 2 * HBYTES + 256 + 1024;
  static constexpr int HSTRIDE = HBYTES, BSTRIDE = B_BYTES;
  static constexpr int TILES_PER_IMAGE = 2;
  static constexpr int DBG = DGRAD ? 32 : 16;
  const ClientRec* recs;
  CnnDims d;

  __device__ void load_b(const TcTile& t, uint32_t sb, uint32_t bar) const {
    if (!DGRAD) {  // W2 shadow [64 co][800 k]: box (64 k, 64 co) per 64-wide K block (the last one zero-filled)
      for (int kb = 0; kb < 13; ++kb) tc::tma_load_2d(sb + kb * 8192, tmap_of(t, TM_W2FS), bar, 64 * kb, 0);
    } else {  // view [64 co][25 tap][32 ci]: box (32 ci, 1 tap, 64 co) per tap
      for (int tap = 0; tap < 25; ++tap) tc::tma_load_3d(sb + tap * 4096, tmap_of(t, TM_W2DS), bar, 0, tap, 0);
    }
  }
  __device__ void load_halo(const TcTile& t, int tile, int grp, uint32_t base, uint32_t bar) const {
    const int r = tile >> 1, x0 = (tile & 1) * 8;
    tc::tma_load_4d(base, tmap_of(t, DGRAD ? TM_DZ2Q1 : TM_A1Q), bar, 32 * grp, x0 - 2, -2, r);
  }
  __device__ void mma_stage(uint32_t hb, uint32_t sb, uint32_t dt, int grp, uint32_t idesc, int = 0) const {
    const uint64_t a0 = tc::sdesc_sw64(hb, 16, 768);
    const uint64_t b0 = !DGRAD ? tc::sdesc_sw128(sb, 16, 1024) : tc::sdesc_sw64(sb, 16, 512);
#pragma unroll
    for (int ky = 0; ky < 5; ++ky)
#pragma unroll
      for (int kx = 0; kx < 5; ++kx) {
        const int tap = ky * 5 + kx;
        const uint32_t ao = (DGRAD ? (4 - ky) * 768 + (4 - kx) * 64 : ky * 768 + kx * 64);
#pragma unroll
        for (int cp = 0; cp < 2; ++cp) {
          uint32_t bo;
          if (!DGRAD) {  // K index = tap*32 + 16 cp: 64-wide block, 32-byte step inside the 128-byte row
            const int kk = 2 * tap + cp;
            bo = (kk >> 2) * 8192 + (kk & 3) * 32;
          } else {  // k rows = co 32 grp + 16 cp .. of tap: 2 atoms of 8 rows per K step
            bo = tap * 4096 + (32 * grp + 16 * cp) * 64;
          }
          tc::mma_bf16_w(dt, tc::dadd(a0, ao + 32 * cp), tc::dadd(b0, bo), idesc, (grp | tap | cp) != 0);
        }
      }
  }
  static constexpr int NCH = (N + 31) / 32;
  struct EpiState {
    const ClientRec* c = nullptr;
    float bias[NCH][16];
  };
  struct Pre {
    uint4 a[NCH][2];
    uint4 i[NCH];
  };
  __device__ void prefetch(const TcTile& t, int tile, int warp, int lane, Pre& p) const {
    if constexpr (DGRAD) {
      const int g = warp >> 2, row = (warp & 3) * 32 + lane;
      const int r = tile >> 1, y = row >> 3, x = (tile & 1) * 8 + (row & 7);
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const int c0 = g * 16 + 32 * j;
        const int64_t o = ((int64_t)r * 256 + y * 16 + x) * W::C1 + c0;
        const uint4* a = reinterpret_cast<const uint4*>((const bf16*)t.c->buf[B_A1] + o);
        p.a[j][0] = a[0];
        p.a[j][1] = a[1];
        p.i[j] = *reinterpret_cast<const uint4*>((const uint8_t*)t.c->buf[B_I1] + o);
      }
    }
  }
  __device__ void epilogue(const TcTile& t, int tile, uint32_t tacc, uint32_t full_bar, uint32_t parity, int warp,
                           int lane, EpiState& st, const Pre&) const {
    const int g = warp >> 2, row = (warp & 3) * 32 + lane;
    const int r = tile >> 1, y = row >> 3, x = (tile & 1) * 8 + (row & 7);
    float a1v[NCH][16];
    int argv[NCH][16];
    if (!DGRAD && st.c != t.c) {
      st.c = t.c;
#pragma unroll
      for (int j = 0; j < NCH; ++j)
#pragma unroll
        for (int q = 0; q < 16; ++q) st.bias[j][q] = t.c->params[d.b2 + g * 16 + 32 * j + q];
    }
    if (DGRAD) {
      Pre p;
      prefetch(t, tile, warp, lane, p);  // operands independent of the MMA: fetch before waiting
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        ld_bf16<16>(reinterpret_cast<const bf16*>(&p.a[j][0]), a1v[j]);
        ld_u8<16>(reinterpret_cast<const uint8_t*>(&p.i[j]), argv[j]);
      }
    }
    tc::mbar_wait(full_bar, parity);
    tc::fence_after();
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c0 = g * 16 + 32 * j;
      float v[16];
      tc::tmem_ld16(tacc + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0, v);
      if (DGRAD) {  // pool-1 backward in the pool-quad layout g1[r][py][px][q][C1] (k_conv1_wgrad_q)
        bf16* g1 = (bf16*)t.c->buf[B_DZC1];
        float out[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int e = 0; e < 16; ++e) out[e] = (argv[j][e] == q && a1v[j][e] > 0.f) ? v[e] : 0.f;
          st_bf16<16>(g1 + (((int64_t)r * 256 + y * 16 + x) * 4 + q) * W::C1 + c0, out);
        }
      } else {  // bias + ReLU + 2x2 max-pool (first max) over lanes (l, l+1, l+8, l+9)
        const int base = lane & ~9;
        float val[16], best[16];
        int arg[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) val[e] = fmaxf(v[e] + st.bias[j][e], 0.f);
        pool_lanes(val, base, base + 1, base + 8, base + 9, best, arg);
        if ((lane & 9) == 0) {
          const int64_t o = ((int64_t)r * 64 + (y >> 1) * 8 + (x >> 1)) * W::C2 + c0;
          st_bf16<16>((bf16*)t.c->buf[B_A2] + o, best);
          st_u8<16>((uint8_t*)t.c->buf[B_I2] + o, arg);
        }
      }
    }
  }
};

// ---------------------------------------------------------------------------
// conv1 fwd (3 -> C1, 32x32 input) + bias + ReLU + 2x2 max-pool, "pool-quad" form.
// One GEMM row per POOLED output (py, px); its 4 pool positions q = (qy, qx)
// become 4 groups of output columns: D[(py,px)][q*C1 + co] = sum over the 6x6
// input window (dy, dx) and ci of xs[2py+dy][2px+dx][ci] * w1q[(dy,dx)][q][co][ci]
// (w1q: common.h, zero outside each q's 5x5 taps).  With the staged input split
// by column parity, the 8 pooled columns of a core matrix read 8 CONSECUTIVE
// 16-byte chunks, so the A operand of the MMA for (dy, dx pair) is a plain
// descriptor into ONE halo buffer (no im2col, no shifted copies): K = 16 =
// (even dx, 8 ci) + (odd dx, 8 ci) at LBO = 160 B, M groups = pooled rows at
// SBO = 640 B.  18 MMAs (M = 128, N = 4 C1, K = 16) per tile; the epilogue pools
// inside a thread (the 4 q columns of a channel), no cross-lane shuffles.
// Tile = 16 pooled rows x 8 pooled columns (2 tiles per image); halo
// [36 rows][2 parities][10 columns][8] = 11.5 KB.
// ---------------------------------------------------------------------------
template <int WQ>
struct QuadConv1 {
  typedef CnnW<WQ> W;
  static constexpr int N = 4 * W::C1;
  static constexpr int NOUT = W::C1;
  static constexpr bool B_MN = false;
  static constexpr int GROUPS = 1;
  static constexpr int HBYTES = 36 * 2 * 10 * 16;
  static constexpr int B_BYTES = 36 * N * 16;  // w1q, [36 K chunks][N][8]
  static constexpr int TMEM_COLS = 2 * N <= 64 ? 64 : 2 * N <= 128 ? 128 : 256;
  static constexpr int SMEM = B_BYTES + 2 * HBYTES + 256 + 1024;
  static constexpr int HSTRIDE = HBYTES, BSTRIDE = B_BYTES;
  static constexpr int TILES_PER_IMAGE = 2;
  static constexpr int NCO = W::C1 >= 32 ? 16 : W::C1;  // channels per epilogue thread
  // (two CTAs per SM measured slower in the light tail: conv1 fwd 22.9 -> 26.3 us per iteration)
  static constexpr int DBG = 48;
  const ClientRec* recs;
  CnnDims d;

  __device__ void load_b(const TcTile& t, uint32_t sb, uint32_t bar) const {
    const uint8_t* w1q = (const uint8_t*)t.c->buf[B_W1P];
    for (int kc = 0; kc < 36; ++kc) tc::bulk_load(sb + kc * N * 16, w1q + kc * N * 16, N * 16, bar);
  }
  __device__ void load_halo(const TcTile& t, int tile, int grp, uint32_t base, uint32_t bar) const {
    tc::tma_load_4d(base, tmap_of(t, TM_XSH), bar, 64 * (tile & 1), 0, 0, tile >> 1);  // 10-pixel runs (160 B)
  }
  __device__ void mma_stage(uint32_t hb, uint32_t sb, uint32_t dt, int grp, uint32_t idesc, int = 0) const {
    const uint64_t a0 = tc::sdesc(hb, 160, 640), b0 = tc::sdesc(sb, N * 16, 128);
#pragma unroll
    for (int dy = 0; dy < 6; ++dy)
#pragma unroll
      for (int dp = 0; dp < 3; ++dp)
        tc::mma_bf16_w(dt, tc::dadd(a0, dy * 320 + dp * 16), tc::dadd(b0, (dy * 3 + dp) * 2 * N * 16), idesc,
                     (dy | dp) != 0);
  }
  struct EpiState {
    const ClientRec* c = nullptr;
    float bias[NCO];
  };
  struct Pre {};
  __device__ void prefetch(const TcTile&, int, int, int, Pre&) const {}
  __device__ void epilogue(const TcTile& t, int tile, uint32_t tacc, uint32_t full_bar, uint32_t parity, int warp,
                           int lane, EpiState& st, const Pre&) const {
    const int g = warp >> 2;
    const bool active = g * NCO < W::C1;  // widths < 1: warps 4-7 idle
    const int r = tile >> 1, row = (warp & 3) * 32 + lane, py = row >> 3, px = (tile & 1) * 8 + (row & 7);
    if (active && st.c != t.c) {
      st.c = t.c;
#pragma unroll
      for (int c = 0; c < NCO; ++c) st.bias[c] = t.c->params[d.b1 + g * NCO + c];
    }
    tc::mbar_wait(full_bar, parity);
    tc::fence_after();
    if (!active) return;
    float v[4 * NCO];
    const uint32_t ta = tacc + ((uint32_t)((warp & 3) * 32) << 16);
    if (NCO == W::C1) {  // the 4 q groups are contiguous columns
#pragma unroll
      for (int k = 0; k < 4 * NCO / 16; ++k) tc::tmem_ld16(ta + 16 * k, *reinterpret_cast<float(*)[16]>(v + 16 * k));
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        tc::tmem_ld16(ta + q * W::C1 + g * NCO, *reinterpret_cast<float(*)[16]>(v + 16 * q));
    }
    float best[NCO];
    int arg[NCO];
#pragma unroll
    for (int c = 0; c < NCO; ++c) {  // bias + ReLU, then the first maximum in q order (strict >)
      float b = fmaxf(v[c] + st.bias[c], 0.f);
      int a = 0;
#pragma unroll
      for (int q = 1; q < 4; ++q) {
        const float x = fmaxf(v[q * NCO + c] + st.bias[c], 0.f);
        if (x > b) {
          b = x;
          a = q;
        }
      }
      best[c] = b;
      arg[c] = a;
    }
    const int64_t o = ((int64_t)r * 256 + py * 16 + px) * W::C1 + g * NCO;
    st_bf16<NCO>((bf16*)t.c->buf[B_A1] + o, best);
    st_u8<NCO>((uint8_t*)t.c->buf[B_I1] + o, arg);
  }
};

// ---------------------------------------------------------------------------
// Persistent kernel.  prefix[] counts TILES per task (rows * TILES_PER_IMAGE);
// CTA b owns global tiles [b*T/grid, (b+1)*T/grid).
// Barriers: b_full / b_empty (client weights), h_full[2] / h_empty[2] (halo
// stages), acc_full[2] / acc_empty[2] (TMEM accumulators).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int next_task(const int* __restrict__ prefix, int ntask, int ti, int g) {
  while (ti + 1 < ntask && __ldg(prefix + ti + 1) <= g) ++ti;
  return ti;
}


template <class Op>
__global__ void __launch_bounds__(kConvThreads, min_blocks<Op>::value)
    k_conv_persistent(const Op op, const Task* __restrict__ tasks, const int* __restrict__ prefix, int ntask) {
  constexpr int D0 = Op::DBG;  // PROTEA_DBG counter block
  constexpr int HST = halo_stages<Op>::value;  // halo ring depth
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sH = smem + Op::BSTRIDE;  // (HBYTES / B_BYTES: the TMA transaction bytes; *STRIDE: the buffer pitch)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sH + HST * Op::HSTRIDE);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6 + 2 * HST);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = __ldg(prefix + ntask);
  const int g0 = (int)((int64_t)blockIdx.x * total / gridDim.x);
  const int g1 = (int)((int64_t)(blockIdx.x + 1) * total / gridDim.x);
  const int ti0 = find_task(prefix, ntask, g0 < total ? g0 : total - 1);
  const uint64_t t_start = threadIdx.x == 0 ? globaltimer() : 0;

  const uint32_t bar0 = tc::smem_u32(bars);
  const uint32_t b_full = bar0, b_empty = bar0 + 8, h_full = bar0 + 16, h_empty = h_full + 8 * HST,
                 acc_full = h_empty + 8 * HST, acc_empty = acc_full + 16;
  if (threadIdx.x == 0) {
    tc::mbar_init(b_full, 1);
    tc::mbar_init(b_empty, 1);
    for (int i = 0; i < HST; ++i) {
      tc::mbar_init(h_full + 8 * i, 1);
      tc::mbar_init(h_empty + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(acc_full + 8 * i, 1);
      tc::mbar_init(acc_empty + 8 * i, 8);
    }
    tc::mbar_fence_init();
  }
  if (warp == 9) tc::tmem_alloc(tc::smem_u32(tmem_slot), Op::TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sb = tc::smem_u32(smem), sh = tc::smem_u32(sH);
  TcTile t;
  t.n_mma = Op::N;
  // the first client's weights were written at least two kernels earlier: load them before the PDL wait
  if (warp == 8 && lane == 0 && g0 < g1) {
    TaskCursor c0;
    c0.init(prefix, ntask, g0);
    t.tk = tasks[c0.ti];
    t.c = op.recs + t.tk.rec;
    tc::mbar_expect_tx(b_full, Op::B_BYTES);
    op.load_b(t, sb, b_full);
  }
  pdl_wait();

  if (warp == 8) {
    if (lane == 0) {  // ---------------- TMA producer
      TaskCursor cur;
      cur.init(prefix, ntask, g0);
      int nb = 0, s = 0;
      for (int g = g0; g < g1; ++g) {
        const bool fresh = cur.advance(prefix, g) || g == g0;
        if (fresh) {  // new client: wait until the MMAs released the previous weights, reload
          t.tk = tasks[cur.ti];
          t.c = op.recs + t.tk.rec;
          if (nb > 0) {  // (the first client's weights were issued before the PDL wait)
            tc::mbar_wait(b_empty, (nb - 1) & 1);
            tc::mbar_expect_tx(b_full, Op::B_BYTES);
            op.load_b(t, sb, b_full);
          }
          ++nb;
        }
        const int tile = g - cur.lo;
        for (int grp = 0; grp < Op::GROUPS; ++grp, ++s) {
          const int buf = s % HST;
          DBG_T0(tw);
          if (s >= HST) tc::mbar_wait(h_empty + 8 * buf, ((s / HST) - 1) & 1);
          DBG_ADD(D0 + 0, tw);
          DBG_T0(ti);
          tc::mbar_expect_tx(h_full + 8 * buf, Op::HBYTES);
          op.load_halo(t, tile, grp, sh + buf * Op::HSTRIDE, h_full + 8 * buf);
          DBG_ADD(D0 + 1, ti);
        }
      }
    }
  } else if (warp == 9) {
    {  // ---------------- MMA issuer (whole warp, elected lane issues)
      const uint32_t idesc = tc::idesc_bf16(128, Op::N, false, Op::B_MN);
      TaskCursor cur;
      cur.init(prefix, ntask, g0);
      int nb = 0, s = 0, i = 0;
      for (int g = g0; g < g1; ++g, ++i) {
        if (cur.advance(prefix, g) || g == g0) {
          if (nb > 0) tc::commit_w(b_empty);  // completes when every MMA issued so far (old weights) is done
          DBG_T0(tb);
          tc::mbar_wait(b_full, nb & 1);
          DBG_ADD(D0 + 6, tb);
          tc::fence_after();
          ++nb;
        }
        const int acc = i & 1;
        DBG_T0(ta0);
        if (i >= 2) tc::mbar_wait(acc_empty + 8 * acc, ((i >> 1) - 1) & 1);
        DBG_ADD(D0 + 2, ta0);
        tc::fence_after();
        for (int grp = 0; grp < Op::GROUPS; ++grp, ++s) {
          const int buf = s % HST;
          DBG_T0(tf);
          tc::mbar_wait(h_full + 8 * buf, (s / HST) & 1);
          DBG_ADD(D0 + 3, tf);
          DBG_T0(tm);
          tc::fence_after();
          op.mma_stage(sh + buf * Op::HSTRIDE, sb, tmem + acc * Op::N, grp, idesc, g - cur.lo);
          tc::commit_w(h_empty + 8 * buf);
          DBG_ADD(D0 + 4, tm);
        }
        tc::commit_w(acc_full + 8 * acc);
      }
    }
    __syncwarp();
  } else if (g0 < g1) {  // ---------------- epilogue warps 0-7 (next tile's operands prefetched)
    typename Op::EpiState st;
    typename Op::Pre pc, pn;
    TaskCursor cur, nxt;
    cur.init(prefix, ntask, g0);
    nxt = cur;
    t.tk = tasks[cur.ti];
    t.c = op.recs + t.tk.rec;
    TcTile tn = t;
    if (xprefetch<Op>::value) op.prefetch(t, g0 - cur.lo, warp, lane, pc);
    int i = 0;
    for (int g = g0; g < g1; ++g, ++i) {
      if (g + 1 < g1) {
        if (nxt.advance(prefix, g + 1)) {
          tn.tk = tasks[nxt.ti];
          tn.c = op.recs + tn.tk.rec;
        }
        if (xprefetch<Op>::value) op.prefetch(tn, g + 1 - nxt.lo, warp, lane, pn);
      }
      const int acc = i & 1;
      DBG_T0(te);
      op.epilogue(t, g - cur.lo, tmem + acc * Op::N, acc_full + 8 * acc, (i >> 1) & 1, warp, lane, st, pc);
      if (warp == 0) DBG_ADD(D0 + 5, te);
      if (PROTEA_DBG && i == 0 && warp == 0 && lane == 0)  // kernel start -> first tile's epilogue done
        atomicAdd(&g_dbg[D0 + 7], (unsigned long long)(globaltimer() - t_start));
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(acc_empty + 8 * acc);
      t = tn;
      cur = nxt;
      pc = pn;
    }
  }
  pdl_trigger();  // main work done: let the next kernel's CTAs start on the SMs this grid frees
  tc::fence_before();
  __syncthreads();
  if (warp == 9) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, Op::TMEM_COLS);
  }
  if (PROTEA_DBG && threadIdx.x == 0) atomicAdd(&g_dbg[D0 + 8], (unsigned long long)(globaltimer() - t_start));
  if (threadIdx.x == 0 && g1 > g0) {  // K9: split this CTA's duration over its clients by tile count
    const uint64_t dt = globaltimer() - t_start;
    int ti = ti0, lo = g0;
    while (lo < g1) {
      const int hi = min(g1, __ldg(prefix + ti + 1));
      const ClientRec* c = op.recs + tasks[ti].rec;
      if (c->sm_ns) atomicAdd((unsigned long long*)c->sm_ns, (unsigned long long)(dt * (hi - lo) / (g1 - g0)));
      lo = hi;
      ++ti;
    }
  }
}

// ---------------------------------------------------------------------------
// conv1 wgrad (width 1, C1 = 32) in pool-quad form.  dz1 is nonzero only at the
// pool window's argmax, so conv2 dgrad stores it per POOLED pixel p as
// g1[p][q][co] (q = 2qy+qx the window position).  Then
//   D[(q,co)][(dy,dx,ci)] = sum_p g1[p][q][co] * xs[2py+dy][2px+dx][ci]     (one GEMM, K = pooled pixels)
//   dW1[co][ky][kx][ci]   = sum_q D[(q,co)][(ky+qy, kx+qx, ci)]            (fold in the epilogue)
//   db1[co]               = sum_q D[(q,co)][(2+qy, 2+qx, 3)]               (staged channel 3 = 1 in the image)
// Work item = (client, split of w1q_ips(rows) images);
// sub-tile = (image, column half) = 128 pooled pixels.  Per K step (16 pooled
// pixels = 2 pooled rows): 6 MMAs (one per dy), M = 128 (q, co), N = 48 (dx, ci).
// A = g1 sub-tile by TMA (two 64-row boxes, 128-byte swizzle, MN-major);
// B = 6 x-shifted copies (one per dx) of the staged rows [36 Y][8 X'][8 ci],
// MN-major without swizzle (core matrix = 8 ci x 8 pooled columns, LBO = next
// pooled row = 256 B, SBO = next dx copy).  TMEM: D at column dy*48 + dx*8 + ci.
// The epilogue folds through shared memory and writes the split's partial
// [76][C1]; the client's last split sums the partials in split order and
// applies SGD to the master and the pool-quad shadow (conv1_reduce_update).
// Persistent: one CTA per SM walks a contiguous range of work items.
// ---------------------------------------------------------------------------
constexpr int kW1GBytes = 2 * 128 * 128;                // g1 sub-tile: 128 (q,co) x 128 pooled px bf16
constexpr int kW1XCopy = 36 * 8 * 16;                   // one dx copy [36][8][8] bf16
constexpr int kW1Stage = kW1GBytes + 6 * kW1XCopy;      // 60416 = 59 x 1024
constexpr int kW1Fold = 4 * 76 * 32 * 4;                // fold buffer S[q][76][32] fp32
constexpr int kW1Stages = 3;                            // TMA ring depth (3 x 59 KB + fold: 216 KB)
constexpr int kW1Smem = kW1Stages * kW1Stage + kW1Fold + 256 + 1024;

__global__ void __launch_bounds__(kConvThreads, 1)
    k_conv1_wgrad_q(const ClientRec* __restrict__ recs, const Task* __restrict__ tasks,
                    const int* __restrict__ prefix, int ntask, int64_t off_w, int64_t off_b, float lr) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  float* S = reinterpret_cast<float*>(smem + kW1Stages * kW1Stage);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kW1Stages * kW1Stage + kW1Fold);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = __ldg(prefix + ntask);
  const int g0 = (int)((int64_t)blockIdx.x * total / gridDim.x);
  const int g1 = (int)((int64_t)(blockIdx.x + 1) * total / gridDim.x);
  const int ti0 = find_task(prefix, ntask, g0 < total ? g0 : total - 1);
  const uint64_t t_start = threadIdx.x == 0 ? globaltimer() : 0;
  const uint32_t bar0 = tc::smem_u32(bars);
  const uint32_t full = bar0, empty = bar0 + 8 * kW1Stages, acc_full = bar0 + 16 * kW1Stages, acc_empty = acc_full + 8;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kW1Stages; ++i) {
      tc::mbar_init(full + 8 * i, 1);
      tc::mbar_init(empty + 8 * i, 1);
    }
    tc::mbar_init(acc_full, 1);
    tc::mbar_init(acc_empty, 8);
    tc::mbar_fence_init();
  }
  if (warp == 9) tc::tmem_alloc(tc::smem_u32(tmem_slot), 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sb = tc::smem_u32(smem);
  pdl_wait();

  if (warp == 8) {
    if (lane == 0) {  // ---------------- TMA producer
      int ti = ti0, s = 0;
      for (int g = g0; g < g1; ++g) {
        ti = next_task(prefix, ntask, ti, g);
        TcTile t;
        t.tk = tasks[ti];
        t.c = recs + t.tk.rec;
        const int ips = w1q_ips(t.tk.rows), r0 = ips * (g - __ldg(prefix + ti)), nsub = 2 * min(ips, t.tk.rows - r0);
        for (int sub = 0; sub < nsub; ++sub, ++s) {
          const int buf = s % kW1Stages, r = r0 + (sub >> 1), h = sub & 1;
          const uint32_t gb = sb + buf * kW1Stage;
          if (s >= kW1Stages) tc::mbar_wait(empty + 8 * buf, ((s / kW1Stages) - 1) & 1);
          tc::mbar_expect_tx(full + 8 * buf, kW1Stage);
          tc::tma_load_4d(gb, tmap_of(t, TM_G), full + 8 * buf, 0, 8 * h, 0, r);
          tc::tma_load_4d(gb + kW1GBytes / 2, tmap_of(t, TM_G), full + 8 * buf, 64, 8 * h, 0, r);
          for (int dx = 0; dx < 6; ++dx)
            tc::tma_load_4d(gb + kW1GBytes + dx * kW1XCopy, tmap_of(t, TM_XSW), full + 8 * buf,
                            8 * (8 * h + (dx >> 1)), dx & 1, 0, r);
        }
      }
    }
  } else if (warp == 9) {
    {  // ---------------- MMA issuer (whole warp, elected lane issues)
      const uint32_t idesc = tc::idesc_bf16(128, 48, true, true);
      int ti = ti0, s = 0, i = 0;
      for (int g = g0; g < g1; ++g, ++i) {
        ti = next_task(prefix, ntask, ti, g);
        const int rows = __ldg(&tasks[ti].rows), ips = w1q_ips(rows);
        const int r0 = ips * (g - __ldg(prefix + ti)), nsub = 2 * min(ips, rows - r0);
        if (i >= 1) tc::mbar_wait(acc_empty, (i - 1) & 1);
        tc::fence_after();
        for (int sub = 0; sub < nsub; ++sub, ++s) {
          const int buf = s % kW1Stages;
          const uint32_t gb = sb + buf * kW1Stage;
          tc::mbar_wait(full + 8 * buf, (s / kW1Stages) & 1);
          tc::fence_after();
          const uint64_t a0 = tc::sdesc_sw128(gb, kW1GBytes / 2, 1024), b0 = tc::sdesc(gb + kW1GBytes, 256, kW1XCopy);
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
#pragma unroll
            for (int dy = 0; dy < 6; ++dy)
              tc::mma_bf16_w(tmem + dy * 48, tc::dadd(a0, 2048 * ks), tc::dadd(b0, (4 * ks + dy) * 128), idesc,
                           (sub | ks) != 0);
          tc::commit_w(empty + 8 * buf);
        }
        tc::commit_w(acc_full);
      }
    }
    __syncwarp();
  } else {  // ---------------- epilogue warps 0-7: warp w holds q = w % 4, ky in [0,3) (w < 4) or [3,5)
    const int q = warp & 3, qy = q >> 1, qx = q & 1, ky0 = warp < 4 ? 0 : 3, ky1 = warp < 4 ? 3 : 5;
    const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16);
    int ti = ti0, i = 0;
    for (int g = g0; g < g1; ++g, ++i) {
      ti = next_task(prefix, ntask, ti, g);
      const ClientRec* c = recs + tasks[ti].rec;
      const int split = g - __ldg(prefix + ti);
      tc::mbar_wait(acc_full, i & 1);
      tc::fence_after();
      float* Sq = S + q * 76 * 32;
      for (int ky = ky0; ky < ky1; ++ky) {
        float v[48];
        const uint32_t col = ta + (uint32_t)((ky + qy) * 48);
#pragma unroll
        for (int k = 0; k < 3; ++k) tc::tmem_ld16(col + 16 * k, *reinterpret_cast<float(*)[16]>(v + 16 * k));
#pragma unroll
        for (int kx = 0; kx < 5; ++kx)
#pragma unroll
          for (int ci = 0; ci < 3; ++ci)
            Sq[((ky * 5 + kx) * 3 + ci) * 32 + lane] = qx ? v[(kx + 1) * 8 + ci] : v[kx * 8 + ci];
        if (ky == 2) Sq[75 * 32 + lane] = qx ? v[3 * 8 + 3] : v[2 * 8 + 3];
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(acc_empty);  // TMEM drained: the next item's MMAs may start
      tc::named_sync(1, 256);
      // partials in dz2 (free from conv2 wgrad's end to the next fc1 dgrad): B_WSP may still hold conv2's
      // partials for their deferred reduce (k_conv2_wgrad_reduce on the side stream)
      float* part = (float*)c->buf[B_DZ2] + (int64_t)split * 76 * 32;
      for (int e = threadIdx.x; e < 76 * 32; e += 256)
        part[e] = ((S[e] + S[2432 + e]) + S[2 * 2432 + e]) + S[3 * 2432 + e];
      // publish this split's partial (arrival counter stats[9])
      __threadfence();
      tc::named_sync(1, 256);
      if (threadIdx.x == 0) atomicAdd(reinterpret_cast<int*>(c->stats) + 9, 1);
    }
    // Split reduce, distributed (as in k_conv2_wgrad_halo): split i of a client (of n) sums slice i of
    // the 76 x C1 partial elements over all splits in split order and applies SGD to it.  It runs after
    // ALL of this CTA's items (the client's other splits live on co-resident CTAs: no deadlock); the
    // last slice to finish resets the counters (stats[9] arrivals, stats[11] slices done).
    TaskCursor rc;
    rc.init(prefix, ntask, g0 < total ? g0 : total - 1);
    for (int g = g0; g < g1; ++g) {
      rc.advance(prefix, g);
      const ClientRec* c = recs + tasks[rc.ti].rec;
      const int splits = cdiv(tasks[rc.ti].rows, w1q_ips(tasks[rc.ti].rows)), item = g - rc.lo;
      int* arrive = reinterpret_cast<int*>(c->stats) + 9;
      int* done = reinterpret_cast<int*>(c->stats) + 11;
      if (threadIdx.x == 0)
        while (atomicAdd(arrive, 0) < splits) __nanosleep(128);
      tc::named_sync(1, 256);
      __threadfence();
      const int e_lo = item * 2432 / splits, e_hi = (item + 1) * 2432 / splits;
      for (int e = e_lo + threadIdx.x; e < e_hi; e += 256)
        conv1_reduce_update(c, splits, 32, off_w, off_b, lr, e, B_DZ2);
      tc::named_sync(1, 256);
      if (threadIdx.x == 0 && atomicAdd(done, 1) == splits - 1) {  // last slice: reset for the next step
        *arrive = 0;
        *done = 0;
      }
    }
  }
  pdl_trigger();  // main work done: let the next kernel's CTAs start on the SMs this grid frees
  tc::fence_before();
  __syncthreads();
  if (warp == 9) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
  if (threadIdx.x == 0 && g1 > g0) {  // K9: split this CTA's duration over its clients by item count
    const uint64_t dt = globaltimer() - t_start;
    int ti = ti0, lo = g0;
    while (lo < g1) {
      const int hi = min(g1, __ldg(prefix + ti + 1));
      const ClientRec* c = recs + tasks[ti].rec;
      if (c->sm_ns) atomicAdd((unsigned long long*)c->sm_ns, (unsigned long long)(dt * (hi - lo) / (g1 - g0)));
      lo = hi;
      ++ti;
    }
  }
}

// ---------------------------------------------------------------------------
// conv2 wgrad (width 1: C1 = 32, C2 = 64) + SGD, single-halo form.  D[m = (tap, ci)][co] =
// sum_p a1[p + tap][ci] dz2[p][co] over the client's output pixels p; ALL 7 M tiles (800
// weights + bias row) accumulate side by side in TMEM (7 x 64 columns).
// Sub-step = 16 output rows x 8 columns (one image half): ONE TMA box brings the a1 halo
// [20 rows][12 px][32 ci] (64-byte swizzle, 15 KB) and one the dz2 tile [16][8][64 co]
// (128-byte swizzle).  Every tap's A operand is a descriptor INTO the halo: the swizzle
// is a function of the absolute shared-memory address, so a start shifted by whole
// 64-byte pixel rows needs no base offset (verified on B200: tools/swz_test.cu).
// MN-major SW64: an atom = 32 channels x 8 consecutive pixels of a halo row; K groups
// (output rows) at SBO = 768 B (one halo row); M tiles j < 5 = taps (ky 0..3, kx = j) at
// LBO = 768, tile 5 = taps (4, kx 0..3) at LBO = 64 (one pixel), tile 6 = tap (4, 4) +
// the bias "ones" block (a constant halo-shaped region after the halo, LBO = 15 KB).
// Work item = (client, split of 8 images = kWgradChunkPx pixels[, M tile]): with ng = 7
// (light iterations) each M tile of a split is its own item.  A client whose batch is
// one split updates the weights straight from TMEM; otherwise every item stores its
// rows of the split's partial [C2][804], and after its CTA's last item each item sums
// one slice of the elements over the splits in split order and applies SGD to the fp32
// master and the bf16 shadow (distributed, balanced reduce; counters stats[8], stats[10]).
// Persistent: one CTA per SM, contiguous item ranges, 3-stage TMA ring.
// ---------------------------------------------------------------------------
constexpr int kW2Halo = 20 * 12 * 64;                   // a1 halo [20][12][32] bf16
constexpr int kW2Dz = 16 * 8 * 128;                     // dz2 [16][8][64] bf16
constexpr int kW2Stage = 2 * kW2Halo + kW2Dz;           // halo + ones block + dz2 = 46 KB
constexpr int kW2Stages = 4;
constexpr int kW2Pad = 16384;  // M tile 6's unused atoms 2-3 read (ignored rows) past the last stage
constexpr int kW2Smem = kW2Stages * kW2Stage + kW2Pad + 256 + 1024;
constexpr int kW2N = 25 * 32 + 1;                        // weight rows + bias row
constexpr int kW2NP = 804;                               // partial row stride (float4-aligned)

__device__ __forceinline__ int w2_row(int j, int row) {  // weight row of TMEM lane `row` in M tile j (-1: none)
  const int atom = row >> 5, ci = row & 31;
  if (j < 5) return (atom * 5 + j) * 32 + ci;
  if (j == 5) return (20 + atom) * 32 + ci;
  if (atom == 0) return 24 * 32 + ci;
  return (atom == 1 && ci == 0) ? 800 : -1;
}

__global__ void __launch_bounds__(kConvThreads, 1)
    k_conv2_wgrad_halo(const ClientRec* __restrict__ recs, const Task* __restrict__ tasks,
                       const int* __restrict__ prefix, int ntask, CnnDims d, float lr, int ng, int defer_reduce) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kW2Stages * kW2Stage + kW2Pad);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kW2Stages + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = __ldg(prefix + ntask);
  const int g0 = (int)((int64_t)blockIdx.x * total / gridDim.x);
  const int g1 = (int)((int64_t)(blockIdx.x + 1) * total / gridDim.x);
  const uint64_t t_start = threadIdx.x == 0 ? globaltimer() : 0;
  const uint32_t bar0 = tc::smem_u32(bars);
  const uint32_t full = bar0, empty = bar0 + 8 * kW2Stages, acc_full = bar0 + 16 * kW2Stages, acc_empty = acc_full + 8;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kW2Stages; ++i) {
      tc::mbar_init(full + 8 * i, 1);
      tc::mbar_init(empty + 8 * i, 1);
    }
    tc::mbar_init(acc_full, 1);
    tc::mbar_init(acc_empty, 8);
    tc::mbar_fence_init();
  }
  // the bias "ones" block of each stage: 1.0 at channel 0 of every 64-byte pixel row; 64-byte
  // swizzle on absolute addresses: logical chunk 0 of the row at byte a sits in chunk (a >> 7) & 3
  for (int i = threadIdx.x; i < kW2Stages * (kW2Halo / 16); i += blockDim.x) {
    const int st = i / (kW2Halo / 16), k = i - st * (kW2Halo / 16);
    const uint32_t off = st * kW2Stage + kW2Halo + 16 * k;
    reinterpret_cast<uint4*>(smem + off)[0] =
        ((off >> 4) & 3) == ((off >> 7) & 3) ? make_uint4(0x3F80u, 0, 0, 0) : make_uint4(0, 0, 0, 0);
  }
  tc::fence_proxy_async();
  if (warp == 9) tc::tmem_alloc(tc::smem_u32(tmem_slot), 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sb = tc::smem_u32(smem);
  TaskCursor cur;
  cur.init(prefix, ntask, g0 < total ? g0 : total - 1);
  pdl_wait();

  if (warp == 8) {
    if (lane == 0) {  // ---------------- TMA producer: per image half, the a1 halo + the dz2 tile
      TcTile t;
      int s = 0;
      for (int g = g0; g < g1; ++g) {
        if (cur.advance(prefix, g) || g == g0) {
          t.tk = tasks[cur.ti];
          t.c = recs + t.tk.rec;
        }
        const int item = g - cur.lo, r0 = 8 * (item / ng), nsub = 2 * min(8, t.tk.rows - r0);
        for (int sub = 0; sub < nsub; ++sub, ++s) {
          const int buf = s % kW2Stages, r = r0 + (sub >> 1), x0 = 8 * (sub & 1);
          const uint32_t base = sb + buf * kW2Stage;
          DBG_T0(tw);
          if (s >= kW2Stages) tc::mbar_wait(empty + 8 * buf, ((s / kW2Stages) - 1) & 1);
          DBG_ADD(0, tw);
          DBG_T0(ti);
          tc::mbar_expect_tx(full + 8 * buf, kW2Halo + kW2Dz);
          tc::tma_load_4d(base, tmap_of(t, TM_A1Q), full + 8 * buf, 0, x0 - 2, -2, r);
          tc::tma_load_4d(base + 2 * kW2Halo, tmap_of(t, TM_DZ2Q), full + 8 * buf, 0, x0, 0, r);
          DBG_ADD(1, ti);
        }
      }
    }
  } else if (warp == 9) {
    {  // ---------------- MMA issuer (whole warp, elected lane issues): 8 K steps x 7 M tiles per half
      const uint32_t idesc = tc::idesc_bf16(128, 64, true, true);
      const uint64_t a_ky = tc::sdesc_sw64(sb, 768, 768), a_kx = tc::sdesc_sw64(sb, 64, 768),
                     a_1 = tc::sdesc_sw64(sb, kW2Halo, 768);
      const uint64_t b0 = tc::sdesc_sw128(sb + 2 * kW2Halo, 16, 1024);
      int s = 0, i = 0;
      for (int g = g0; g < g1; ++g, ++i) {
        cur.advance(prefix, g);
        const int item = g - cur.lo, grp = item % ng, r0 = 8 * (item / ng);
        const int nsub = 2 * min(8, __ldg(&tasks[cur.ti].rows) - r0);
        DBG_T0(ta0);
        if (i >= 1) tc::mbar_wait(acc_empty, (i - 1) & 1);
        DBG_ADD(2, ta0);
        tc::fence_after();
        for (int sub = 0; sub < nsub; ++sub, ++s) {
          const int buf = s % kW2Stages;
          const uint32_t so = buf * kW2Stage;
          DBG_T0(tf);
          tc::mbar_wait(full + 8 * buf, (s / kW2Stages) & 1);
          DBG_ADD(3, tf);
          DBG_T0(tm);
          tc::fence_after();
          if (ng == 1) {
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              const uint64_t db = tc::dadd(b0, so + 2048 * ks);
              const uint32_t acc = (sub | ks) != 0, row = so + 2 * ks * 768;
#pragma unroll
              for (int j = 0; j < 5; ++j) tc::mma_bf16_w(tmem + 64 * j, tc::dadd(a_ky, row + 64 * j), db, idesc, acc);
              tc::mma_bf16_w(tmem + 64 * 5, tc::dadd(a_kx, row + 4 * 768), db, idesc, acc);
              tc::mma_bf16_w(tmem + 64 * 6, tc::dadd(a_1, row + 4 * 768 + 4 * 64), db, idesc, acc);
            }
          } else {  // one M tile
            const uint64_t a = grp < 5 ? tc::dadd(a_ky, so + 64 * grp)
                                       : grp == 5 ? tc::dadd(a_kx, so + 4 * 768) : tc::dadd(a_1, so + 4 * 768 + 256);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
              tc::mma_bf16_w(tmem + 64 * grp, tc::dadd(a, 2 * ks * 768), tc::dadd(b0, so + 2048 * ks), idesc,
                             (sub | ks) != 0);
          }
          tc::commit_w(empty + 8 * buf);
          DBG_ADD(4, tm);
        }
        tc::commit_w(acc_full);
      }
    }
    __syncwarp();
  } else {  // ---------------- epilogue warps 0-7: lanes (warp % 4) * 32.., columns 32 (warp / 4)..
    const int row = (warp & 3) * 32 + lane, cb = (warp >> 2) * 32;
    const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const int Kw = 800;
    int i = 0;
    for (int g = g0; g < g1; ++g, ++i) {
      cur.advance(prefix, g);
      const Task tk = tasks[cur.ti];
      const ClientRec* c = recs + tk.rec;
      const int item = g - cur.lo, split = item / ng, grp = item % ng, splits = (tk.rows + 7) / 8;
      float* P = c->params;
      bf16* S = (bf16*)c->buf[B_WSH];
      float* part = (float*)c->buf[B_WSP] + (int64_t)split * 64 * kW2NP;
      DBG_T0(te);
      tc::mbar_wait(acc_full, i & 1);
      if (warp == 0) DBG_ADD(5, te);
      DBG_T0(td);
      tc::fence_after();
#pragma unroll 1
      for (int j = ng == 1 ? 0 : grp; j < (ng == 1 ? 7 : grp + 1); ++j) {
        float v[32];
        tc::tmem_ld16(ta + 64 * j + cb, *reinterpret_cast<float(*)[16]>(v));
        tc::tmem_ld16(ta + 64 * j + cb + 16, *reinterpret_cast<float(*)[16]>(v + 16));
        const int m = w2_row(j, row);
        if (m < 0) continue;
        if (splits == 1) {  // whole batch in this item: SGD straight from the accumulator
          if (m == Kw) {
#pragma unroll
            for (int q = 0; q < 32; ++q) P[d.b2 + cb + q] -= lr * v[q];
          } else {
            float w[32];
#pragma unroll
            for (int q = 0; q < 32; ++q) w[q] = P[d.w2 + (int64_t)(cb + q) * Kw + m];
#pragma unroll
            for (int q = 0; q < 32; ++q) {
              const int64_t idx = d.w2 + (int64_t)(cb + q) * Kw + m;
              const float nw = w[q] - lr * v[q];
              P[idx] = nw;
              S[idx] = __float2bfloat16_rn(nw);
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q) part[(int64_t)(cb + q) * kW2NP + m] = v[q];
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(acc_empty);  // TMEM drained: the next item's MMAs may start
      if (warp == 0) DBG_ADD(6, td);
      DBG_T0(tr);
      if (splits > 1 && !defer_reduce) {  // publish this item's partial (arrival counter stats[8])
        __threadfence();
        tc::named_sync(1, 256);
        if (threadIdx.x == 0) atomicAdd(reinterpret_cast<int*>(c->stats) + 8, 1);
      }
      if (warp == 0) DBG_ADD(7, tr);
    }
    // Split reduce, distributed: item i of a client (of n = splits * ng) sums slice i of the client's
    // 64 x 804 partial elements in split order and applies SGD to it.  It runs after ALL of this CTA's
    // items, so waiting for the client's other items (other CTAs, all co-resident: grid <= #SMs) cannot
    // deadlock; the last slice to finish resets the counters (stats[8] arrivals, stats[10] slices done).
    DBG_T0(tsr);
    TaskCursor rc;
    rc.init(prefix, ntask, g0 < total ? g0 : total - 1);
    for (int g = g0; g < (defer_reduce ? g0 : g1); ++g) {  // deferred: k_conv2_wgrad_reduce
      rc.advance(prefix, g);
      const Task tk = tasks[rc.ti];
      const int splits = (tk.rows + 7) / 8, nitem = splits * ng, item = g - rc.lo;
      if (splits == 1) continue;
      const ClientRec* c = recs + tk.rec;
      int* arrive = reinterpret_cast<int*>(c->stats) + 8;
      int* done = reinterpret_cast<int*>(c->stats) + 10;
      if (threadIdx.x == 0)
        while (atomicAdd(arrive, 0) < nitem) __nanosleep(256);
      tc::named_sync(1, 256);
      __threadfence();
      float* P = c->params;
      bf16* S = (bf16*)c->buf[B_WSH];
      const float4* pt = (const float4*)c->buf[B_WSP];
      constexpr int Q = kW2NP / 4, NE = 64 * Q;  // float4 chunks per split
      const int e_lo = (int)((int64_t)item * NE / nitem), e_hi = (int)((int64_t)(item + 1) * NE / nitem);
#pragma unroll 2
      for (int e = e_lo + threadIdx.x; e < e_hi; e += 256) {
        const int co = e / Q, m0 = 4 * (e - co * Q);
        const int64_t idx = d.w2 + (int64_t)co * 800 + m0;
        float4 w = m0 < 800 ? *reinterpret_cast<const float4*>(P + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 q[8];  // splits <= 8 (B <= 64): every load in flight at once, summed in split order
#pragma unroll
        for (int sp = 0; sp < 8; ++sp)
          if (sp < splits) q[sp] = __ldcg(pt + (int64_t)sp * NE + e);
        float4 gs = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int sp = 0; sp < 8; ++sp)
          if (sp < splits) gs.x += q[sp].x, gs.y += q[sp].y, gs.z += q[sp].z, gs.w += q[sp].w;
        if (m0 < 800) {
          w.x -= lr * gs.x, w.y -= lr * gs.y, w.z -= lr * gs.z, w.w -= lr * gs.w;
          *reinterpret_cast<float4*>(P + idx) = w;
          const __nv_bfloat162 h0 = __floats2bfloat162_rn(w.x, w.y), h1 = __floats2bfloat162_rn(w.z, w.w);
          *reinterpret_cast<uint2*>(S + idx) =
              make_uint2(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1));
        } else if (m0 == 800) {
          P[d.b2 + co] -= lr * gs.x;
        }
      }
      tc::named_sync(1, 256);
      if (threadIdx.x == 0 && atomicAdd(done, 1) == nitem - 1) {  // last slice: reset for the next step
        *arrive = 0;
        *done = 0;
      }
    }
    if (warp == 0) DBG_ADD(9, tsr);
  }
  pdl_trigger();  // main work done: let the next kernel's CTAs start on the SMs this grid frees
  tc::fence_before();
  __syncthreads();
  if (warp == 9) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
  if (PROTEA_DBG && threadIdx.x == 0) atomicAdd(&g_dbg[8], (unsigned long long)(globaltimer() - t_start));
  if (threadIdx.x == 0 && g1 > g0) {  // K9: split this CTA's duration over its clients by item count
    const uint64_t dt = globaltimer() - t_start;
    int ti = find_task(prefix, ntask, g0), lo = g0;
    while (lo < g1) {
      const int hi = min(g1, __ldg(prefix + ti + 1));
      const ClientRec* c = recs + tasks[ti].rec;
      if (c->sm_ns) atomicAdd((unsigned long long*)c->sm_ns, (unsigned long long)(dt * (hi - lo) / (g1 - g0)));
      lo = hi;
      ++ti;
    }
  }
}

// conv2 wgrad split reduce as its own launch (the deferred form of k_conv2_wgrad_halo's in-kernel
// reduce): block (x, task) sums float4 chunk x of the client's [C2][804] partials over its splits in
// split order and applies SGD to the fp32 master and the bf16 shadow.  Launched on the side stream
// after the wgrad, joined before the group's next conv2 fwd (the next reader of the weights).
__global__ void __launch_bounds__(256) k_conv2_wgrad_reduce(const ClientRec* __restrict__ recs,
                                                            const Task* __restrict__ tasks, CnnDims d, float lr) {
  const Task tk = tasks[blockIdx.y];
  const int splits = (tk.rows + 7) / 8;
  if (splits == 1) return;  // updated from TMEM by the wgrad kernel
  const ClientRec* c = recs + tk.rec;
  constexpr int Q = kW2NP / 4, NE = 64 * Q;
  const int e = blockIdx.x * 256 + threadIdx.x;
  if (e >= NE) return;
  float* P = c->params;
  bf16* S = (bf16*)c->buf[B_WSH];
  const float4* pt = (const float4*)c->buf[B_WSP];
  const int co = e / Q, m0 = 4 * (e - co * Q);
  const int64_t idx = d.w2 + (int64_t)co * 800 + m0;
  float4 w = m0 < 800 ? *reinterpret_cast<const float4*>(P + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 q[8];
#pragma unroll
  for (int sp = 0; sp < 8; ++sp)
    if (sp < splits) q[sp] = __ldcg(pt + (int64_t)sp * NE + e);
  float4 gs = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int sp = 0; sp < 8; ++sp)
    if (sp < splits) gs.x += q[sp].x, gs.y += q[sp].y, gs.z += q[sp].z, gs.w += q[sp].w;
  if (m0 < 800) {
    w.x -= lr * gs.x, w.y -= lr * gs.y, w.z -= lr * gs.z, w.w -= lr * gs.w;
    *reinterpret_cast<float4*>(P + idx) = w;
    const __nv_bfloat162 h0 = __floats2bfloat162_rn(w.x, w.y), h1 = __floats2bfloat162_rn(w.z, w.w);
    *reinterpret_cast<uint2*>(S + idx) =
        make_uint2(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1));
  } else if (m0 == 800) {
    P[d.b2 + co] -= lr * gs.x;
  }
}

}  // namespace protea
