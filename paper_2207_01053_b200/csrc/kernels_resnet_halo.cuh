// kernels_resnet_halo.cuh — ResNet-8 stride-1 3x3 convolutions (layers 1, 2, 4, 6: C -> C channels at
// C x C... H = 32 / 16 / 8 for C = 16 / 32 / 64) as "halo" implicit GEMMs on the persistent tcgen05
// kernel k_conv_persistent (kernels_conv.cuh), fwd and dgrad.
//
// The cp.async-gathered form (kernels_resnet_tc.cuh) issues one 16-byte copy per (pixel, tap, 8
// channels): ~1,300 instructions per 128 x 64 K block, instruction-issue bound.  Here
// a tile is 16 output rows x 8 columns of one image (M row m = y * 8 + x; 8x8 images fill rows 0-63 and
// leave 64-127 unused) and its whole input is ONE TMA box: the halo [18 rows][10 px][C ch] with the
// swizzle whose width is one pixel's C channels (SW32 / SW64 / SW128 for C = 16 / 32 / 64); the conv's
// zero padding is the TMA's out-of-bounds fill.  The A operand of tap (ky, kx) is a K-major descriptor
// into that box shifted by ky halo rows + kx pixels (8-row core groups = 8 pixels of one halo row,
// SBO = one halo row; the swizzle follows absolute shared-memory addresses, tools/swz_test.cu), so a
// tile costs one TMA and 9 x C/16 MMAs (M = 128, N = C, K = 16).
//   fwd   D[p][co] = sum_{ky,kx,ci} in[p + (ky-1, kx-1)][ci] W[co][ky][kx][ci]
//         B = the client's 9 weight taps [co][ci] (K-major), resident while the CTA stays on the client;
//         epilogue + bias (+ identity / option-A residual), ReLU -> bf16 (as RTcFwd)
//   dgrad D[p][ci] = sum_{ky,kx,co} dout[p - (ky-1, kx-1)][co] W[co][ky][kx][ci]
//         same weight boxes read MN-major (K = co rows, N = ci), flipped taps into the dout halo;
//         epilogue (+ identity add) x ReLU mask of the stored activation -> bf16 (as RTcDgrad)
// Same arithmetic as the gathered kernels (fp32 accumulation of the same products; only the order of
// the K accumulation differs), parity against the oracle in tests/test_gpu_tc.py / test_gpu_parity.py.
#pragma once
#include "kernels_conv.cuh"
#include "kernels_resnet_tc.cuh"

namespace protea {

// per-client tensor maps of the ResNet-8 halo kernels (same 19-slot array as the CNN's TmapId)
enum RTmapId : int {
  RTM_IN1 = 0, RTM_IN2, RTM_IN4, RTM_IN6,  // fwd input halos of layers 1, 2, 4, 6: box (C, 10, 18, 1)
  RTM_DO1, RTM_DO2, RTM_DO4, RTM_DO6,      // dgrad dout halos of layers 1, 2, 4, 6
  RTM_W1, RTM_W2, RTM_W4, RTM_W6,          // weight shadow of layers 1, 2, 4, 6 [co][9][ci]: box (C, 1, C)
  RTM_WD1, RTM_WD2, RTM_WD4, RTM_WD6,      // wgrad dout halos of layers 1, 2, 4, 6: box (C, 8, 18, 1)
  RTM_IN3, RTM_IN5,                        // stride-2 fwd input of layers 3, 5 as pixel pairs: box (Cin, 9, 33, 1)
  RTM_W3, RTM_W5,                          // their weight taps [co][9][ci]: box (Cin, 1, Cout)
  RTM_DO3, RTM_DO5,                        // stride-2 dgrad dout halos of layers 3, 5: box (Cout, 9, 17, 1)
  RTM_WD3, RTM_WD5,                        // stride-2 wgrad dout tiles of layers 3, 5: box (Cout, 8, 16, 1)
  RTM_IN0,                                 // conv0: the staged input [r][32][32 x 8] as 160-byte halo rows: box (80, 19, 1)
  RTM_W0,                                  // conv0: the padded weight taps [16][9][8]: box (8, 1, 16)
  RTM_WD0,                                 // conv0 wgrad dout halo (dz0, 16 ch): box (16, 8, 18, 1)
  RTM_COUNT
};
static_assert((int)RTM_COUNT <= kTmapSlots, "ResNet-8 maps exceed the per-client map array");

__device__ __forceinline__ uint64_t sdesc_swc(uint32_t saddr, uint32_t sbo, int rb, uint32_t lbo = 16) {
  // swizzle width = rb bytes (one pixel's channels): 32 -> SW32 (6), 64 -> SW64 (4), 128 -> SW128 (2)
  const uint64_t lt = rb == 32 ? 6 : rb == 64 ? 4 : 2;
  return tc::sdesc(saddr, lbo, sbo) | (lt << 61);
}

template <int C, bool DGRAD>
struct RHalo {
  static constexpr int H = C == 16 ? 32 : C == 32 ? 16 : 8, W = H;
  static constexpr int N = C, NOUT = C;
  static constexpr bool B_MN = DGRAD;
  static constexpr int GROUPS = 1;
  static constexpr int RB = 2 * C;       // bytes of one pixel = the swizzle width
  static constexpr int PITCH = 10 * RB;  // one halo row
  static constexpr int HALO = 18 * PITCH;
  static constexpr int HBYTES = HALO, HSTRIDE = (HALO + 1023) & ~1023;  // TMA bytes / 1024-aligned buffer pitch
  static constexpr int TAPB = C * C * 2;  // one tap's weights [co][ci]
  static constexpr int B_BYTES = 9 * TAPB, BSTRIDE = (B_BYTES + 1023) & ~1023;
  static constexpr int TMEM_COLS = 2 * N <= 32 ? 32 : 2 * N <= 64 ? 64 : 128;
  static constexpr int HSTAGES = C == 16 ? 6 : C == 32 ? 4 : 3;  // halo ring: TMA latency over small tiles
  static constexpr int SMEM = BSTRIDE + HSTAGES * HSTRIDE + 256 + 1024;
  static constexpr int TX = W / 8, TY = (H + 15) / 16, TILES_PER_IMAGE = TX * TY;
  static constexpr int NC = N / 2;                  // accumulator columns per epilogue warp group
  static constexpr int CW = NC < 16 ? NC : 16, NCH = NC / CW;  // tcgen05.ld width, loads per thread
  static constexpr int MIN_BLOCKS = C == 64 ? 1 : C == 32 ? 2 : 3;  // resident CTAs per SM (C = 64: smem)
  static constexpr int DBG = 0;
  const ClientRec* recs;
  int in_tm, w_tm;       // tensor maps: input (fwd) / dout (dgrad) halo, weight taps
  int out_buf;           // fwd: activation out; dgrad: input gradient out
  int res_buf, res_mode, Cres;  // fwd residual (1 identity, 2 option A); dgrad add (1 identity)
  int mask_buf;          // dgrad: ReLU mask = the stored activation of the layer input
  int64_t b_off;         // fwd: bias offset in params

  __device__ void load_b(const TcTile& t, uint32_t sb, uint32_t bar) const {
    for (int tap = 0; tap < 9; ++tap) tc::tma_load_3d(sb + tap * TAPB, tmap_of(t, w_tm), bar, 0, tap, 0);
  }
  __device__ void load_halo(const TcTile& t, int tile, int, uint32_t base, uint32_t bar) const {
    const int r = tile / TILES_PER_IMAGE, q = tile - r * TILES_PER_IMAGE;
    const int y0 = (q / TX) * 16, x0 = (q % TX) * 8;
    tc::tma_load_4d(base, tmap_of(t, in_tm), bar, 0, x0 - 1, y0 - 1, r);
  }
  __device__ void mma_stage(uint32_t hb, uint32_t sb, uint32_t dt, int, uint32_t idesc, int = 0) const {
    const uint64_t a0 = sdesc_swc(hb, PITCH, RB), b0 = sdesc_swc(sb, 8 * RB, RB);
#pragma unroll
    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) {
        const int tap = ky * 3 + kx;
        const uint32_t ao = DGRAD ? (2 - ky) * PITCH + (2 - kx) * RB : ky * PITCH + kx * RB;
#pragma unroll
        for (int ks = 0; ks < C / 16; ++ks) {
          // fwd: K = ci, 16 channels = +32 B inside the pixel row; dgrad: K = co rows, 16 rows = 2 core groups
          const uint32_t bo = tap * TAPB + (DGRAD ? ks * 16 * RB : ks * 32);
          tc::mma_bf16_w(dt, tc::dadd(a0, ao + 32 * ks), tc::dadd(b0, bo), idesc, (tap | ks) != 0);
        }
      }
  }
  struct EpiState {
    const ClientRec* c = nullptr;
    float bias[NCH][CW];
  };
  // the epilogue's global operands (fwd: residual; dgrad: identity add and ReLU mask) are loaded one tile
  // ahead (k_conv_persistent, XPF): their latency overlaps the previous tile's epilogue
  static constexpr bool XPF = true;
  static constexpr int NV = CW / 8;  // 16-byte vectors per chunk
  struct Pre {
    uint4 p[NCH][NV];
    uint4 m[DGRAD ? NCH : 1][NV];
  };
  __device__ void prefetch(const TcTile& t, int tile, int warp, int lane, Pre& pr) const {
    const int g = warp >> 2, row = (warp & 3) * 32 + lane;
    const int r = tile / TILES_PER_IMAGE, q = tile - r * TILES_PER_IMAGE;
    const int y = (q / TX) * 16 + (row >> 3), x = (q % TX) * 8 + (row & 7);
    const bool valid = y < H;
    const int64_t pix = ((int64_t)r * H + y) * W + x;
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c0 = g * NC + CW * j;
      const bf16* src = nullptr;
      if (valid && res_mode == 1)
        src = (const bf16*)t.c->buf[res_buf] + pix * C + c0;
      else if (valid && !DGRAD && res_mode == 2 && c0 < Cres)
        src = (const bf16*)t.c->buf[res_buf] + (((int64_t)r * 2 * H + 2 * y) * 2 * W + 2 * x) * Cres + c0;
#pragma unroll
      for (int v = 0; v < NV; ++v) pr.p[j][v] = src ? reinterpret_cast<const uint4*>(src)[v] : make_uint4(0, 0, 0, 0);
      if constexpr (DGRAD) {
#pragma unroll
        for (int v = 0; v < NV; ++v)
          pr.m[j][v] = valid ? reinterpret_cast<const uint4*>((const bf16*)t.c->buf[mask_buf] + pix * C + c0)[v]
                             : make_uint4(0, 0, 0, 0);
      }
    }
  }
  __device__ void epilogue(const TcTile& t, int tile, uint32_t tacc, uint32_t full_bar, uint32_t parity, int warp,
                           int lane, EpiState& st, const Pre& pr) const {
    const int g = warp >> 2, row = (warp & 3) * 32 + lane;  // warp group g: columns [g NC, (g + 1) NC)
    const int r = tile / TILES_PER_IMAGE, q = tile - r * TILES_PER_IMAGE;
    const int y = (q / TX) * 16 + (row >> 3), x = (q % TX) * 8 + (row & 7);
    const bool valid = y < H;
    const int64_t pix = ((int64_t)r * H + y) * W + x;
    if (!DGRAD && st.c != t.c) {
      st.c = t.c;
#pragma unroll
      for (int j = 0; j < NCH; ++j)
#pragma unroll
        for (int e = 0; e < CW; ++e) st.bias[j][e] = t.c->params[b_off + g * NC + CW * j + e];
    }
    tc::mbar_wait(full_bar, parity);
    tc::fence_after();
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c0 = g * NC + CW * j;
      float v[CW], pre[CW];
      const uint32_t ta = tacc + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0;
      if constexpr (CW == 16) tc::tmem_ld16(ta, v); else tc::tmem_ld8(ta, v);
      if (!valid) continue;
      ld_bf16<CW>(reinterpret_cast<const bf16*>(&pr.p[j][0]), pre);
      float o[CW];
      if constexpr (!DGRAD) {
#pragma unroll
        for (int e = 0; e < CW; ++e) o[e] = fmaxf(v[e] + st.bias[j][e] + pre[e], 0.f);
      } else {
        float msk[CW];
        ld_bf16<CW>(reinterpret_cast<const bf16*>(&pr.m[j][0]), msk);
#pragma unroll
        for (int e = 0; e < CW; ++e) o[e] = msk[e] > 0.f ? v[e] + pre[e] : 0.f;
      }
      st_bf16<CW>((bf16*)t.c->buf[out_buf] + pix * C + c0, o);
    }
  }
};

// ---------------------------------------------------------------------------
// conv0 fwd (3 -> 16 ch at 32x32) on the staged input xs [r][32][32][8] bf16 (channels 3-7 zero) and the
// padded weights w0p [16][9][8] (B_R_W0P).  A pixel is 16 bytes, so the halo [18 (+1) rows][10 px][8 ch] is
// ONE 2-D TMA box of 160-byte rows (x viewed as 256 elements per image row; the conv's zero padding is
// the out-of-bounds fill, also at element -8).  A is K-major without swizzle: core matrix = 8 pixels of
// a halo row (16-byte rows), SBO = one halo row (160 B), LBO = 16 B = the NEXT pixel, so one K = 16 MMA
// covers two horizontally adjacent taps (ky, kx) and (ky, kx + 1).  B = [ky][kx 0..3][co 16][ci 8] with
// the (ky, 3) blocks zero: 6 MMAs (M = 128, N = 16, K = 16) per 16 x 8 tile.  Epilogue bias + ReLU -> a0.
// ---------------------------------------------------------------------------
struct RHalo0 {
  static constexpr int H = 32, W = 32, N = 16, NOUT = 16;
  static constexpr bool B_MN = false;
  static constexpr int GROUPS = 1;
  // 19 halo rows: the pseudo-tap (2, 3) reads one pixel past row 17 (times a zero weight), which must be
  // finite data, not stale shared memory (NaN x 0 = NaN)
  static constexpr int PITCH = 160, HBYTES = 19 * PITCH, HSTRIDE = 3072;
  static constexpr int B_BYTES = 12 * 256, BSTRIDE = 12 * 256;  // 9 taps + 3 zero blocks, all by TMA
  static constexpr int TMEM_COLS = 32;
  static constexpr int HSTAGES = 6;
  static constexpr int SMEM = BSTRIDE + HSTAGES * HSTRIDE + 256 + 1024;
  static constexpr int TX = 4, TILES_PER_IMAGE = 8;
  static constexpr int NC = 8;  // accumulator columns per epilogue warp group
  static constexpr int MIN_BLOCKS = 3;
  static constexpr int DBG = 0;
  const ClientRec* recs;
  int out_buf;
  int64_t b_off;

  __device__ void load_b(const TcTile& t, uint32_t sb, uint32_t bar) const {
    // block (ky, kx) <- tap ky * 3 + kx; the (ky, 3) blocks are the map's out-of-bounds tap 9: the TMA's zero
    // fill (generic-proxy stores here would not be ordered before the barrier's completion)
    for (int ky = 0; ky < 3; ++ky)
      for (int kx = 0; kx < 4; ++kx)
        tc::tma_load_3d(sb + (ky * 4 + kx) * 256, tmap_of(t, RTM_W0), bar, 0, kx < 3 ? ky * 3 + kx : 9, 0);
  }
  __device__ void load_halo(const TcTile& t, int tile, int, uint32_t base, uint32_t bar) const {
    const int r = tile >> 3, q = tile & 7, y0 = (q >> 2) * 16, x0 = (q & 3) * 8;
    tc::tma_load_3d(base, tmap_of(t, RTM_IN0), bar, 8 * (x0 - 1), y0 - 1, r);
  }
  __device__ void mma_stage(uint32_t hb, uint32_t sb, uint32_t dt, int, uint32_t idesc, int = 0) const {
    const uint64_t a0 = tc::sdesc(hb, 16, PITCH), b0 = tc::sdesc(sb, 256, 128);
#pragma unroll
    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
      for (int p = 0; p < 2; ++p)
        tc::mma_bf16_w(dt, tc::dadd(a0, ky * PITCH + 32 * p), tc::dadd(b0, (ky * 4 + 2 * p) * 256), idesc,
                       (ky | p) != 0);
  }
  struct EpiState {
    const ClientRec* c = nullptr;
    float bias[NC];
  };
  struct Pre {};
  __device__ void prefetch(const TcTile&, int, int, int, Pre&) const {}
  __device__ void epilogue(const TcTile& t, int tile, uint32_t tacc, uint32_t full_bar, uint32_t parity, int warp,
                           int lane, EpiState& st, const Pre&) const {
    const int g = warp >> 2, row = (warp & 3) * 32 + lane;
    const int r = tile >> 3, q = tile & 7;
    const int y = (q >> 2) * 16 + (row >> 3), x = (q & 3) * 8 + (row & 7);
    if (st.c != t.c) {
      st.c = t.c;
#pragma unroll
      for (int e = 0; e < NC; ++e) st.bias[e] = t.c->params[b_off + g * NC + e];
    }
    tc::mbar_wait(full_bar, parity);
    tc::fence_after();
    float v[NC], o[NC];
    tc::tmem_ld8(tacc + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(g * NC), v);
#pragma unroll
    for (int e = 0; e < NC; ++e) o[e] = fmaxf(v[e] + st.bias[e], 0.f);
    st_bf16<NC>((bf16*)t.c->buf[out_buf] + (((int64_t)r * H + y) * W + x) * 16 + g * NC, o);
  }
};

// ---------------------------------------------------------------------------
// Stride-2 fwd (layers 3: 16 -> 32 ch, 32x32 -> 16x16; 5: 32 -> 64 ch, 16x16 -> 8x8).  Output tile =
// 16 x 8 output pixels (8x8 outputs: rows 8-15 unused).  Output (yo, xo) reads input (2yo+ky-1,
// 2xo+kx-1): the input rows are viewed as pixel PAIRS [H][W/2][2 Cin], so one TMA box of Cin channels
// at channel offset 0 / Cin is the plane of even / odd input columns; two boxes [33 rows][9 pairs][Cin]
// per tile.  Tap (ky, kx) reads plane kx == 1 ? even : odd at pair offset kx == 2, starting at row ky,
// with 8-row core groups = 8 consecutive xo (consecutive pairs: RB bytes apart) and SBO = TWO plane
// rows (yo -> 2 yo).  Epilogue bias + ReLU (the block's residual is added by its second conv).
// ---------------------------------------------------------------------------
template <int CIN>
struct RHaloS2 {
  static constexpr int H = CIN == 16 ? 32 : 16, W = H, HO = H / 2, WO = W / 2;
  static constexpr int N = 2 * CIN, NOUT = N, COUT = N;
  static constexpr bool B_MN = false;
  static constexpr int GROUPS = 1;
  static constexpr int RB = 2 * CIN;            // bytes of one input pixel = the swizzle width
  static constexpr int PP = 9 * RB;             // one plane row (9 pixels of one parity)
  static constexpr int PLANE = 33 * PP;         // TMA bytes of one plane
  static constexpr int PSTRIDE = (PLANE + 1023) & ~1023;
  static constexpr int HBYTES = 2 * PLANE, HSTRIDE = 2 * PSTRIDE;
  static constexpr int TAPB = COUT * CIN * 2;   // one tap's weights [co][ci]
  static constexpr int B_BYTES = 9 * TAPB, BSTRIDE = (B_BYTES + 1023) & ~1023;
  static constexpr int TMEM_COLS = 2 * N <= 64 ? 64 : 128;
  static constexpr int HSTAGES = CIN == 16 ? 4 : 3;
  static constexpr int SMEM = BSTRIDE + HSTAGES * HSTRIDE + 256 + 1024;
  static constexpr int TX = WO / 8, TY = (HO + 15) / 16, TILES_PER_IMAGE = TX * TY;
  static constexpr int NC = N / 2, NCH = NC / 16;
  static constexpr int MIN_BLOCKS = CIN == 16 ? 2 : 1;  // (CIN = 32: shared memory)
  static constexpr int DBG = 0;
  const ClientRec* recs;
  int in_tm, w_tm, out_buf;
  int64_t b_off;

  __device__ void load_b(const TcTile& t, uint32_t sb, uint32_t bar) const {
    for (int tap = 0; tap < 9; ++tap) tc::tma_load_3d(sb + tap * TAPB, tmap_of(t, w_tm), bar, 0, tap, 0);
  }
  __device__ void load_halo(const TcTile& t, int tile, int, uint32_t base, uint32_t bar) const {
    const int r = tile / TILES_PER_IMAGE, q = tile - r * TILES_PER_IMAGE;
    const int y0 = (q / TX) * 16, x0 = (q % TX) * 8;
    tc::tma_load_4d(base, tmap_of(t, in_tm), bar, 0, x0, 2 * y0 - 1, r);                // even columns 2 x0 ..
    tc::tma_load_4d(base + PSTRIDE, tmap_of(t, in_tm), bar, CIN, x0 - 1, 2 * y0 - 1, r);  // odd columns 2 x0 - 1 ..
  }
  __device__ void mma_stage(uint32_t hb, uint32_t sb, uint32_t dt, int, uint32_t idesc, int = 0) const {
    const uint64_t a0 = sdesc_swc(hb, 2 * PP, RB), b0 = sdesc_swc(sb, 8 * RB, RB);
#pragma unroll
    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) {
        const int tap = ky * 3 + kx;
        const uint32_t ao = (kx == 1 ? 0 : PSTRIDE) + ky * PP + (kx == 2 ? RB : 0);
#pragma unroll
        for (int ks = 0; ks < CIN / 16; ++ks)
          tc::mma_bf16_w(dt, tc::dadd(a0, ao + 32 * ks), tc::dadd(b0, tap * TAPB + 32 * ks), idesc, (tap | ks) != 0);
      }
  }
  struct EpiState {
    const ClientRec* c = nullptr;
    float bias[NCH][16];
  };
  struct Pre {};
  __device__ void prefetch(const TcTile&, int, int, int, Pre&) const {}
  __device__ void epilogue(const TcTile& t, int tile, uint32_t tacc, uint32_t full_bar, uint32_t parity, int warp,
                           int lane, EpiState& st, const Pre&) const {
    const int g = warp >> 2, row = (warp & 3) * 32 + lane;
    const int r = tile / TILES_PER_IMAGE, q = tile - r * TILES_PER_IMAGE;
    const int y = (q / TX) * 16 + (row >> 3), x = (q % TX) * 8 + (row & 7);
    if (st.c != t.c) {
      st.c = t.c;
#pragma unroll
      for (int j = 0; j < NCH; ++j)
#pragma unroll
        for (int e = 0; e < 16; ++e) st.bias[j][e] = t.c->params[b_off + g * NC + 16 * j + e];
    }
    tc::mbar_wait(full_bar, parity);
    tc::fence_after();
    const int64_t pix = ((int64_t)r * HO + y) * WO + x;
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c0 = g * NC + 16 * j;
      float v[16];
      tc::tmem_ld16(tacc + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0, v);
      if (y >= HO) continue;
      float o[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) o[e] = fmaxf(v[e] + st.bias[j][e], 0.f);
      st_bf16<16>((bf16*)t.c->buf[out_buf] + pix * COUT + c0, o);
    }
  }
};

// ---------------------------------------------------------------------------
// Stride-2 dgrad (layers 3, 5): dIn[y][x] = sum over the taps with y + 1 - ky and x + 1 - kx even of
// dout[(y + 1 - ky) / 2][(x + 1 - kx) / 2] W[.][ky][kx].  The input pixels split into 4 parity classes
// (py, px) = (y & 1, x & 1); inside a class every row of a tile uses the SAME taps: ky = 1 for py = 0,
// ky in {0, 2} for py = 1 (likewise kx), at dout offset (py + 1 - ky) / 2 in {0, 1}.  A tile = 16 x 8
// pixels (i, j) of one class (y = 2i + py, x = 2j + px); its A operands are descriptors into one dout
// halo [17 rows][9 px][Cout] (offsets 0 / +1 row / +1 pixel; rows past the image are the TMA's zero
// fill): 1, 2, 2 or 4 taps x Cout / 16 MMAs per tile.  B = the weight taps read MN-major (K = co,
// N = ci), as RHalo<dgrad>.  Epilogue (+ option-A shortcut gradient at even (y, x), channels < Cin)
// x ReLU mask -> bf16 (as RTcDgrad, add_mode 2).
// ---------------------------------------------------------------------------
template <int CIN>
struct RHaloS2D {
  static constexpr int H = CIN == 16 ? 32 : 16, W = H, HO = H / 2, WO = W / 2, COUT = 2 * CIN;
  static constexpr int N = CIN, NOUT = N;
  static constexpr bool B_MN = true;
  static constexpr int GROUPS = 1;
  static constexpr int RBO = 2 * COUT, RBI = 2 * CIN;  // dout pixel bytes (A swizzle), weight row bytes (B)
  static constexpr int PITCH = 9 * RBO;
  static constexpr int HALO = 17 * PITCH;
  static constexpr int HBYTES = HALO, HSTRIDE = (HALO + 1023) & ~1023;
  static constexpr int TAPB = COUT * CIN * 2;
  static constexpr int B_BYTES = 9 * TAPB, BSTRIDE = (B_BYTES + 1023) & ~1023;
  static constexpr int TMEM_COLS = 2 * N <= 32 ? 32 : 64;
  static constexpr int HSTAGES = CIN == 16 ? 4 : 3;
  static constexpr int SMEM = BSTRIDE + HSTAGES * HSTRIDE + 256 + 1024;
  static constexpr int TX = WO / 8, TY = (HO + 15) / 16, TPC = TX * TY, TILES_PER_IMAGE = 4 * TPC;
  static constexpr int NC = N / 2, CW = NC < 16 ? NC : 16, NCH = NC / CW;
  static constexpr int MIN_BLOCKS = 2;
  static constexpr int DBG = 0;
  const ClientRec* recs;
  int in_tm, w_tm, out_buf, add_buf, Cadd, mask_buf;

  __device__ void load_b(const TcTile& t, uint32_t sb, uint32_t bar) const {
    for (int tap = 0; tap < 9; ++tap) tc::tma_load_3d(sb + tap * TAPB, tmap_of(t, w_tm), bar, 0, tap, 0);
  }
  __device__ static void coords(int tile, int& r, int& cls, int& i0, int& j0) {
    r = tile / TILES_PER_IMAGE;
    const int q = tile - r * TILES_PER_IMAGE;
    cls = q / TPC;
    i0 = ((q % TPC) / TX) * 16;
    j0 = (q % TX) * 8;
  }
  __device__ void load_halo(const TcTile& t, int tile, int, uint32_t base, uint32_t bar) const {
    int r, cls, i0, j0;
    coords(tile, r, cls, i0, j0);
    tc::tma_load_4d(base, tmap_of(t, in_tm), bar, 0, j0, i0, r);
  }
  __device__ void mma_stage(uint32_t hb, uint32_t sb, uint32_t dt, int, uint32_t idesc, int tile = 0) const {
    int r, cls, i0, j0;
    coords(tile, r, cls, i0, j0);
    const int py = cls >> 1, px = cls & 1;
    const uint64_t a0 = sdesc_swc(hb, PITCH, RBO), b0 = sdesc_swc(sb, 8 * RBI, RBI);
    bool acc = false;
#pragma unroll
    for (int ky = 0; ky < 3; ++ky) {
      if ((ky == 1) != (py == 0)) continue;  // py = 0: ky = 1; py = 1: ky = 0, 2
      const int dyo = (py + 1 - ky) / 2;
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) {
        if ((kx == 1) != (px == 0)) continue;
        const int dxo = (px + 1 - kx) / 2, tap = ky * 3 + kx;
#pragma unroll
        for (int ks = 0; ks < COUT / 16; ++ks) {
          tc::mma_bf16_w(dt, tc::dadd(a0, dyo * PITCH + dxo * RBO + 32 * ks), tc::dadd(b0, tap * TAPB + ks * 16 * RBI),
                         idesc, acc);
          acc = true;
        }
      }
    }
  }
  struct EpiState {};
  static constexpr bool XPF = true;  // mask / shortcut gradient loaded one tile ahead (as RHalo)
  static constexpr int NV = CW / 8;
  struct Pre {
    uint4 p[NCH][NV], m[NCH][NV];
  };
  __device__ void prefetch(const TcTile& t, int tile, int warp, int lane, Pre& pr) const {
    const int g = warp >> 2, row = (warp & 3) * 32 + lane;
    int r, cls, i0, j0;
    coords(tile, r, cls, i0, j0);
    const int i = i0 + (row >> 3), j = j0 + (row & 7), y = 2 * i + (cls >> 1), x = 2 * j + (cls & 1);
    const bool valid = i < HO;
    const int64_t pix = ((int64_t)r * H + y) * W + x;
#pragma unroll
    for (int jj = 0; jj < NCH; ++jj) {
      const int c0 = g * NC + CW * jj;
      const bool add = valid && cls == 0 && c0 < Cadd;  // option-A shortcut gradient at even (y, x)
      const uint4* ps = reinterpret_cast<const uint4*>((const bf16*)t.c->buf[add_buf] +
                                                       (((int64_t)r * HO + i) * WO + j) * Cadd + c0);
      const uint4* ms = reinterpret_cast<const uint4*>((const bf16*)t.c->buf[mask_buf] + pix * CIN + c0);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        pr.p[jj][v] = add ? ps[v] : make_uint4(0, 0, 0, 0);
        pr.m[jj][v] = valid ? ms[v] : make_uint4(0, 0, 0, 0);
      }
    }
  }
  __device__ void epilogue(const TcTile& t, int tile, uint32_t tacc, uint32_t full_bar, uint32_t parity, int warp,
                           int lane, EpiState&, const Pre& pr) const {
    const int g = warp >> 2, row = (warp & 3) * 32 + lane;
    int r, cls, i0, j0;
    coords(tile, r, cls, i0, j0);
    const int i = i0 + (row >> 3), j = j0 + (row & 7), y = 2 * i + (cls >> 1), x = 2 * j + (cls & 1);
    const bool valid = i < HO;
    const int64_t pix = ((int64_t)r * H + y) * W + x;
    tc::mbar_wait(full_bar, parity);
    tc::fence_after();
#pragma unroll
    for (int jj = 0; jj < NCH; ++jj) {
      const int c0 = g * NC + CW * jj;
      float v[CW];
      const uint32_t ta = tacc + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0;
      if constexpr (CW == 16) tc::tmem_ld16(ta, v); else tc::tmem_ld8(ta, v);
      if (!valid) continue;
      float o[CW], pre[CW], msk[CW];
      ld_bf16<CW>(reinterpret_cast<const bf16*>(&pr.p[jj][0]), pre);
      ld_bf16<CW>(reinterpret_cast<const bf16*>(&pr.m[jj][0]), msk);
#pragma unroll
      for (int e = 0; e < CW; ++e) o[e] = msk[e] > 0.f ? v[e] + pre[e] : 0.f;
      st_bf16<CW>((bf16*)t.c->buf[out_buf] + pix * CIN + c0, o);
    }
  }
};

// ---------------------------------------------------------------------------
// Weight gradient of the same layers, one work item per 2048-pixel split of a client (the split
// partials of kernels_resnet_tc.cuh RTcWgrad, summed in split order + SGD by k_reduce_multi_v4):
//   dW[co][ky][kx][ci] = sum_p in[p + (ky-1, kx-1)][ci] dout[p][co],   K = the split's pixels
// Stride 1 (RWgHalo, RWgHalo0): per 16 x 8 tile the TMA brings the input halo (as the fwd) and the dout
// tile WITH one halo row above and below [18][8][C].  Summing over the input pixels q of the tile instead
// of the output pixels: dW[ky][kx] = sum_q in[q + (0, kx-1)][ci] dout[q - (ky-1, 0)][co]; the tiles'
// input rows partition the image, so every (q, ky) pair is counted once (dout rows -1 / H are the
// TMA's zero fill).  A = the input rows of the tile read MN-major: M = (kx, ci), the three kx "atoms"
// ONE pixel (RB bytes) apart (LBO = RB: the same bytes serve the three column shifts), K = pixels
// (8 per halo row, SBO = one halo row).  B = the dout halo read MN-major with N = (a, co): atom a = the
// dout rows shifted by a (LBO = one dout row), i.e. tap row ky = 2 - a.  So ONE MMA covers all nine
// taps (M = 3C <= 128, N = 3C; C = 64: kx 0-1 and kx 2 as two MMAs).  The bias gradient sum_p dout[p][co]
// is one more MMA (N = C, the unshifted atom a = 1) with A = a 128-byte block of bf16 ones (LBO = SBO = 0).
// Accumulators stay in TMEM over the split's tiles (double-buffered across items where TMEM allows);
// the 8 epilogue warps write the partial [co][9 C + 1] rows (row m of the accumulator = (kx, ci):
// consecutive lanes store consecutive weights).
// Warp roles as k_conv_persistent: 0-7 epilogue, 8 TMA producer (lane 0), 9 MMA issuer.
// ---------------------------------------------------------------------------
template <int C>
struct RWgHalo {  // stride 1: C -> C
  typedef RHalo<C, false> G;
  static constexpr int H = G::H, W = G::W, RB = G::RB, PITCH = G::PITCH, TPI = G::TILES_PER_IMAGE;
  static constexpr int COUT = C, CIN = C;
  static constexpr int MH = C == 64 ? 2 : 1;                                 // M = (kx, ci) halves
  static constexpr int NMMA = 3 * COUT;                                      // N = (a, co) of the tap MMAs
  static constexpr int NBLK = 3 * MH;                                        // accumulator blocks (mh, a)
  static constexpr int RBO = 2 * COUT, DBYTES = 144 * RBO;                   // dout halo [18][8][Cout]
  static constexpr int B_LBO = 8 * RBO;                                      // N atoms: one dout row apart
  static constexpr int BIAS_B = 8 * RBO;                                     // the unshifted atom (a = 1)
  static constexpr int HB = G::HSTRIDE, STAGE = HB + ((DBYTES + 1023) & ~1023);
  static constexpr int TX_BYTES = G::HALO + DBYTES;
  static constexpr int STAGES = C == 64 ? 3 : 4;
  static constexpr int COLS = (NBLK + 1) * COUT;                             // + the bias accumulator
  static constexpr int NACC = 2 * COLS <= 512 ? 2 : 1;
  static constexpr int TMEM_COLS = NACC * COLS <= 32 ? 32 : NACC * COLS <= 64 ? 64 : NACC * COLS <= 128 ? 128
                                   : NACC * COLS <= 256 ? 256 : 512;
  static constexpr int SMEM = STAGES * STAGE + 256 + 128 + 1024;
  static constexpr int N_PART = 9 * CIN + 1;                                 // partial row: 9 Cin weights + bias
  __device__ static void load(uint32_t st, const uint8_t* tm, int in_tm, int dout_tm, int tile, uint32_t bar) {
    const int r = tile / TPI, q = tile - r * TPI, y0 = (q / (W / 8)) * 16, x0 = (q % (W / 8)) * 8;
    tc::tma_load_4d(st, tm + 128 * in_tm, bar, 0, x0 - 1, y0 - 1, r);
    tc::tma_load_4d(st + HB, tm + 128 * dout_tm, bar, 0, x0, y0 - 1, r);  // dout rows y0 - 1 .. y0 + 16
  }
  // K step ks = tile pixel rows 2 ks, 2 ks + 1 (halo rows 2 ks + 1, + 2); block (mh, a) at columns (3 mh + a) C
  __device__ static void mma(uint32_t st, uint32_t ta, int ks, bool acc, uint32_t idesc, uint64_t bk) {
    const uint64_t a0 = sdesc_swc(st, PITCH, RB, RB);  // LBO = RB: the kx atoms one pixel apart
#pragma unroll
    for (int mh = 0; mh < MH; ++mh)
      tc::mma_bf16_w(ta + mh * NMMA, tc::dadd(a0, (1 + 2 * ks) * PITCH + mh * 2 * RB), bk, idesc, acc);
  }
  __device__ static bool row_of(int blk, int m, int& n) {  // accumulator row m of block blk -> partial column
    const int mh = blk / 3, ky = 2 - blk % 3, kx = mh * (128 / C) + m / C;
    n = (ky * 3 + kx) * C + m % C;
    return kx < 3;
  }
};

// conv0 (3 -> 16 at 32x32) over RHalo0's 160-byte-row halo of the staged input.  A = the tile's input rows
// read MN-major without swizzle: core matrix = 8 channels of one pixel (16 B) x 8 consecutive pixels (K
// rows, 16 B apart), M groups j at SBO = 16 B = the next pixel (kx = j, j < 3; channels ci < 3 real),
// K groups at LBO = one halo row.  B = the dz0 halo with the tap rows as N atoms, as RWgHalo<16>.
// Partial rows [16][28] (9 x 3 weights + bias).
struct RWgHalo0 {
  static constexpr int COUT = 16, CIN = 3, TPI = 8;
  static constexpr int PITCH = RHalo0::PITCH;
  static constexpr int NMMA = 3 * COUT, NBLK = 3;
  static constexpr int RBO = 2 * COUT, DBYTES = 144 * RBO;
  static constexpr int B_LBO = 8 * RBO, BIAS_B = 8 * RBO;
  static constexpr int HB = 3072, STAGE = HB + ((DBYTES + 1023) & ~1023);
  static constexpr int TX_BYTES = RHalo0::HBYTES + DBYTES;
  static constexpr int STAGES = 6;
  static constexpr int COLS = (NBLK + 1) * COUT;
  static constexpr int NACC = 2;
  static constexpr int TMEM_COLS = 128;
  static constexpr int SMEM = STAGES * STAGE + 256 + 128 + 1024;
  static constexpr int N_PART = 9 * CIN + 1;
  __device__ static void load(uint32_t st, const uint8_t* tm, int in_tm, int dout_tm, int tile, uint32_t bar) {
    const int r = tile >> 3, q = tile & 7, y0 = (q >> 2) * 16, x0 = (q & 3) * 8;
    tc::tma_load_3d(st, tm + 128 * in_tm, bar, 8 * (x0 - 1), y0 - 1, r);
    tc::tma_load_4d(st + HB, tm + 128 * dout_tm, bar, 0, x0, y0 - 1, r);
  }
  __device__ static void mma(uint32_t st, uint32_t ta, int ks, bool acc, uint32_t idesc, uint64_t bk) {
    tc::mma_bf16_w(ta, tc::dadd(tc::sdesc(st, PITCH, 16), (1 + 2 * ks) * PITCH), bk, idesc, acc);
  }
  __device__ static bool row_of(int blk, int m, int& n) {
    const int j = m >> 3, ci = m & 7, ky = 2 - blk;
    n = (ky * 3 + j) * CIN + ci;
    return j < 3 && ci < CIN;
  }
};

template <int CIN>
struct RWgHaloS2 {  // stride 2: CIN -> 2 CIN, over the pixel-pair planes of RHaloS2
  typedef RHaloS2<CIN> G;
  static constexpr int COUT = 2 * CIN, RB = G::RB, PP = G::PP, TPI = G::TILES_PER_IMAGE, HO = G::HO, WO = G::WO;
  static constexpr int NBLK = 6;                                             // (ky, odd plane: kx 0, 2), (ky, even: kx 1)
  static constexpr int NMMA = COUT, B_LBO = 16, BIAS_B = 0;                  // (one N atom: the dout tile itself)
  static constexpr int RBO = 2 * COUT, DBYTES = 128 * RBO;
  static constexpr int HB = G::HSTRIDE, STAGE = HB + ((DBYTES + 1023) & ~1023);
  static constexpr int TX_BYTES = G::HBYTES + DBYTES;
  static constexpr int STAGES = CIN == 16 ? 4 : 2;
  static constexpr int COLS = (NBLK + 1) * COUT;
  static constexpr int NACC = 2 * COLS <= 512 ? 2 : 1;
  static constexpr int TMEM_COLS = 512;
  static constexpr int SMEM = STAGES * STAGE + 256 + 128 + 1024;
  static constexpr int N_PART = 9 * CIN + 1;
  __device__ static void load(uint32_t st, const uint8_t* tm, int in_tm, int dout_tm, int tile, uint32_t bar) {
    const int r = tile / TPI, q = tile - r * TPI, y0 = (q / G::TX) * 16, x0 = (q % G::TX) * 8;
    tc::tma_load_4d(st, tm + 128 * in_tm, bar, 0, x0, 2 * y0 - 1, r);                    // even columns
    tc::tma_load_4d(st + G::PSTRIDE, tm + 128 * in_tm, bar, CIN, x0 - 1, 2 * y0 - 1, r);  // odd columns
    tc::tma_load_4d(st + HB, tm + 128 * dout_tm, bar, 0, x0, y0, r);
  }
  // output rows 2 ks, 2 ks + 1 read plane rows 4 ks + ky (+ 2): SBO = two plane rows
  __device__ static void mma(uint32_t st, uint32_t ta, int ks, bool acc, uint32_t idesc, uint64_t bk) {
    // odd plane: M atoms kx = 0 (pair offset 0) and kx = 2 (the next pair, RB bytes on): LBO = RB;
    // even plane: atom 0 = kx = 1 (the others unused rows)
    const uint64_t ae = sdesc_swc(st, 2 * PP, RB, RB), ao = sdesc_swc(st + G::PSTRIDE, 2 * PP, RB, RB);
#pragma unroll
    for (int ky = 0; ky < 3; ++ky) {
      tc::mma_bf16_w(ta + (2 * ky) * COUT, tc::dadd(ao, (4 * ks + ky) * PP), bk, idesc, acc);
      tc::mma_bf16_w(ta + (2 * ky + 1) * COUT, tc::dadd(ae, (4 * ks + ky) * PP), bk, idesc, acc);
    }
  }
  __device__ static bool row_of(int blk, int m, int& n) {
    const int ky = blk >> 1, a = m / CIN, odd = !(blk & 1);
    const int kx = odd ? (a == 0 ? 0 : a == 1 ? 2 : 3) : (a == 0 ? 1 : 3);
    n = (ky * 3 + kx) * CIN + m % CIN;
    return kx < 3;
  }
};

// Persistent weight-gradient kernel over one geometry P (RWgHalo / RWgHaloS2 / RWgHalo0).
template <class P>
__global__ void __launch_bounds__(kConvThreads, P::TMEM_COLS <= 256 ? 2 : 1)
    k_r8_wgrad_halo(const ClientRec* __restrict__ recs, const Task* __restrict__ tasks, const int* __restrict__ prefix,
                    int ntask, int in_tm, int dout_tm, int layer) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P::STAGES * P::STAGE);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * P::STAGES + 4);
  uint16_t* ones = reinterpret_cast<uint16_t*>(smem + P::STAGES * P::STAGE + 256);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = __ldg(prefix + ntask);
  const int g0 = (int)((int64_t)blockIdx.x * total / gridDim.x);
  const int g1 = (int)((int64_t)(blockIdx.x + 1) * total / gridDim.x);
  const int ti0 = find_task(prefix, ntask, g0 < total ? g0 : total - 1);
  const uint64_t t_start = threadIdx.x == 0 ? globaltimer() : 0;
  const uint32_t bar0 = tc::smem_u32(bars);
  const uint32_t full = bar0, empty = bar0 + 8 * P::STAGES, acc_full = bar0 + 16 * P::STAGES, acc_empty = acc_full + 16;
  if (threadIdx.x == 0) {
    for (int s = 0; s < P::STAGES; ++s) {
      tc::mbar_init(full + 8 * s, 1);
      tc::mbar_init(empty + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(acc_full + 8 * a, 1);
      tc::mbar_init(acc_empty + 8 * a, 8);
    }
    tc::mbar_fence_init();
  }
  if (threadIdx.x < 64) ones[threadIdx.x] = 0x3F80;  // bf16 1.0
  if (warp == 9) tc::tmem_alloc(tc::smem_u32(tmem_slot), P::TMEM_COLS);
  tc::fence_proxy_async();  // the ones block is read by the tensor cores (async proxy)
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sb = tc::smem_u32(smem);
  pdl_wait();

  if (warp == 8) {
    if (lane == 0) {  // ---------------- TMA producer: per tile the input halo / planes and the dout tile
      int s = 0, ti = ti0;
      for (int g = g0; g < g1; ++g) {
        ti = next_task(prefix, ntask, ti, g);
        const Task tk = tasks[ti];
        const ClientRec* c = recs + tk.rec;
        const uint8_t* tm = reinterpret_cast<const uint8_t*>(c->tmaps);
        const int sp = g - __ldg(prefix + ti);
        const int r0 = r8_split_image(layer, tk.rows, sp), r1 = r8_split_image(layer, tk.rows, sp + 1);
        for (int tile = r0 * P::TPI; tile < r1 * P::TPI; ++tile, ++s) {
          const int buf = s % P::STAGES;
          if (s >= P::STAGES) tc::mbar_wait(empty + 8 * buf, ((s / P::STAGES) - 1) & 1);
          tc::mbar_expect_tx(full + 8 * buf, P::TX_BYTES);
          P::load(sb + buf * P::STAGE, tm, in_tm, dout_tm, tile, full + 8 * buf);
        }
      }
    }
  } else if (warp == 9) {  // ---------------- MMA issuer (whole warp, elected lane issues)
    const uint32_t idesc = tc::idesc_bf16(128, P::NMMA, true, true), idesc1 = tc::idesc_bf16(128, P::COUT, false, true);
    const uint64_t d1 = tc::sdesc(tc::smem_u32(ones), 0, 0);
    int s = 0, i = 0, ti = ti0;
    for (int g = g0; g < g1; ++g, ++i) {
      ti = next_task(prefix, ntask, ti, g);
      const int rows = __ldg(&tasks[ti].rows), sp = g - __ldg(prefix + ti);
      const int r0 = r8_split_image(layer, rows, sp), r1 = r8_split_image(layer, rows, sp + 1);
      const int a = P::NACC == 2 ? (i & 1) : 0;
      const uint32_t ta = tmem + a * P::COLS;
      if (P::NACC == 2 ? i >= 2 : i >= 1)
        tc::mbar_wait(acc_empty + 8 * a, (P::NACC == 2 ? (i >> 1) - 1 : i - 1) & 1);
      tc::fence_after();
      for (int tile = r0 * P::TPI; tile < r1 * P::TPI; ++tile, ++s) {
        const int buf = s % P::STAGES;
        const uint32_t st = sb + buf * P::STAGE;
        tc::mbar_wait(full + 8 * buf, (s / P::STAGES) & 1);
        tc::fence_after();
        const bool first = tile == r0 * P::TPI;
        const uint64_t b0 = sdesc_swc(st + P::HB, 8 * P::RBO, P::RBO, P::B_LBO);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {  // 16 pixels = 2 tile rows per K step
          const uint64_t bk = tc::dadd(b0, ks * 16 * P::RBO);
          P::mma(st, ta, ks, !(first && ks == 0), idesc, bk);
          tc::mma_bf16_w(ta + P::NBLK * P::COUT, d1, tc::dadd(bk, P::BIAS_B), idesc1, !(first && ks == 0));
        }
        tc::commit_w(empty + 8 * buf);
      }
      tc::commit_w(acc_full + 8 * a);
    }
    __syncwarp();
  } else {  // ---------------- epilogue warps 0-7: lane quadrant warp % 4 = accumulator rows m
    const int m = (warp & 3) * 32 + lane, half = warp >> 2;
    int i = 0, ti = ti0;
    for (int g = g0; g < g1; ++g, ++i) {
      ti = next_task(prefix, ntask, ti, g);
      const ClientRec* c = recs + tasks[ti].rec;
      const int split = g - __ldg(prefix + ti);
      const int a = P::NACC == 2 ? (i & 1) : 0;
      const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16) + a * P::COLS;
      tc::mbar_wait(acc_full + 8 * a, (P::NACC == 2 ? (i >> 1) : i) & 1);
      tc::fence_after();
      float* part = (float*)c->buf[B_R_WSP] + r8_wsp_off(layer, c->B) + (int64_t)split * P::COUT * P::N_PART;
      // accumulator blocks and the bias block; the two warp groups take alternate co chunks
      // (Cout = 16: warp group 1 idles)
      if (16 * half < P::COUT) {
#pragma unroll
        for (int blk = 0; blk <= P::NBLK; ++blk) {
          const bool bias = blk == P::NBLK;
          int n = 0;
          const bool ok = bias ? m == 0 : P::row_of(blk, m, n);
          if (bias) n = P::N_PART - 1;
#pragma unroll
          for (int cc = 0; cc < (P::COUT + 31) / 32; ++cc) {
            const int c0 = 16 * half + 32 * cc;
            float v[16];
            tc::tmem_ld16(ta + blk * P::COUT + c0, v);
            if (ok) {
#pragma unroll
              for (int e = 0; e < 16; ++e) part[(int64_t)(c0 + e) * P::N_PART + n] = v[e];
            }
          }
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(acc_empty + 8 * a);
    }
  }
  pdl_trigger();
  tc::fence_before();
  __syncthreads();
  if (warp == 9) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, P::TMEM_COLS);
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

}  // namespace protea
