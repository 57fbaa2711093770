// common.h — library-internal types shared by the host runtime and the kernels.
//
// Model table, parameter layout and the per-client arena slot layout
// (DESIGN.md "Arena slot layout").  This is the library's own copy; the
// oracle (oracle/profiler.py) implements the same table independently and the
// CPU tests compare the two byte for byte through protea_client_footprint.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/protea.h"

namespace protea {

constexpr uint64_t kAlign = 256;
inline uint64_t align256(uint64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// One layer of a model, in forward order.  Weights are [out][K] row-major with
// K = k*k*cin (conv, NHWC taps (ky,kx,ci)) or K = in (fc); bias [out] follows.
struct Layer {
  int kind;      // 0 = conv, 1 = fc, 2 = GroupNorm (cin = cout = C; "weights" = gamma [C], "bias" = beta [C])
  int k, stride, pad;
  int cin, cout;
  int hin, win;  // input spatial size (conv)
  int hout, wout;
  int64_t off_w, off_b;  // offsets in the flat parameter vector
  int64_t K() const { return kind == 0 ? (int64_t)k * k * cin : kind == 1 ? cin : 1; }
};

struct ModelDims {
  int arch = 0, width_q = 4, classes = 10, H = 0, W = 0, C = 0;
  int c1 = 0, c2 = 0, f = 0;  // CNN channel counts
  int64_t P = 0;
  std::vector<Layer> layers;
  int64_t in_dim() const { return (int64_t)H * W * C; }
};

bool make_model(const protea_model_desc& d, ModelDims* out, std::string* err);

// FLOPs of one sample's forward + backward pass: 2 * (fwd + wgrad + dgrad MACs),
// no dgrad for the first layer.
uint64_t flops_per_sample(const ModelDims& m);

// Named buffers of one client's slot, in slot order.
enum Buf : int {
  B_PARAMS = 0, B_PERM, B_STATS, B_WSH,
  // MLP
  B_H1, B_DZ1,
  // CNN
  B_A1, B_I1, B_A2, B_I2, B_H, B_DH, B_DZ2, B_DZC1, B_XS, B_W1P, B_WSP,
  // ResNet-8
  B_R_A0, B_R_R1, B_R_O1, B_R_R2, B_R_O2, B_R_R3, B_R_O3, B_R_GAP, B_R_DGAP, B_R_G0, B_R_G1, B_R_G2,
  B_R_W0P,  // bf16 mode: conv0 weights padded to 8 input channels [16][9][8] (tensor-core operand)
  B_R_XS,   // bf16 mode: conv0 input staged as [r][32][32][8] bf16 (read by conv0 fwd and wgrad)
  B_R_WSP,
  // ResNet-18 (GroupNorm, reading R26): conv layer l = 0..16 in forward order (stem, then blocks i = 0..7 as
  // l = 1 + 2i (conv a), 2 + 2i (conv b)); z_l = the conv output, y_l = the activation after GroupNorm (+
  // shortcut) and ReLU
  B_G_Z0,
  B_G_Y0 = B_G_Z0 + 17,
  B_G_ST = B_G_Y0 + 17,  // GroupNorm statistics [b][17 layers][2 groups][mean, rstd] fp32
  B_G_X, B_G_YG, B_G_ZG,  // gradient buffers (the largest activation each)
  B_G_GNP,               // GroupNorm parameter-gradient partials [b][2][512] fp32 (per layer, reused)
  B_G_WSP,               // conv weight-gradient split partials (per layer, reused: max over layers)
  B_COUNT
};
constexpr int kGroups = 2;    // GroupNorm groups (R26)
constexpr int kG_Layers = 17;  // ResNet-18 conv layers

struct SlotLayout {
  uint64_t off[B_COUNT];
  uint64_t size[B_COUNT];
  bool used[B_COUNT];
  uint64_t total;  // = exact HWM of the slot (bump allocator, nothing freed in a round)
};

// Split-K partition of the conv wgrad reductions (pixels per split).
constexpr int kWgradChunkPx = 2048;
// width-1 pool-quad conv1 wgrad (k_conv1_wgrad_q): images per split, a function of the client's own batch
// rows only (client results must not depend on the cohort): 2 for the smallest batches (parallelism in
// the light tail), 4 otherwise (half the per-split epilogues / partials in heavy iterations)
#if defined(__CUDACC__)
__host__ __device__
#endif
inline int w1q_ips(int rows) { return rows >= 16 ? 4 : 2; }
int cnn_conv1_splits(int rows);
int cnn_conv2_splits(int rows);

SlotLayout slot_layout(const ModelDims& m, int batch, int64_t n, int epochs, int elem_bytes);

// Batches larger than kMicroRows rows (§4.3: batch sizes 1024 / 2048) run as micro-clients:
// the batch's rows are cut into ceil(min(B, n) / kMicroRows) chunks, each a full client slot of
// min(kMicroRows, rest) rows that takes its SGD step from the same weights; after the step a merge kernel
// forms w + sum_m (b_m / |beta|) (w_m - w) = w - lr grad(mean over |beta|) (engine.cu).
// The client's slot is the micro slots back to back followed by the merge weights (fp32, P floats).
constexpr int kMicroRows = 64;
constexpr float kMicroLrScale = 1048576.0f;  // micro SGD steps use lr * 2^20 (exact scaling, see engine.cu)
// Exact arena high-water mark of a client (= slot_layout(...).total when min(B, n) <= kMicroRows).
uint64_t client_hwm(const ModelDims& m, int batch, int64_t n, int epochs, int elem_bytes);
inline int micro_count(int batch, int64_t n) {
  const int64_t b = batch < n ? batch : n;
  return b <= kMicroRows ? 1 : (int)((b + kMicroRows - 1) / kMicroRows);
}

// bf16-mode conv1 "pool-quad" weight shadow w1q (buffer B_W1P), DESIGN.md §6:
// [dy 6][dx>>1 3][dx&1 2][n = q*C1 + co][ci 8] bf16, q = 2qy+qx a position of
// the 2x2 pool window and (dy, dx) = (qy+ky, qx+kx) the tap's offset inside the
// 6x6 input window of one pooled output; entry = W1[co][ky][kx][ci] (zero when
// ky or kx is outside 0..4 or ci >= 3).
#if defined(__CUDACC__)
__host__ __device__
#endif
inline int64_t w1q_index(int C1, int dy, int dx, int q, int co, int ci) {
  return ((int64_t)((dy * 3 + (dx >> 1)) * 2 + (dx & 1)) * (4 * C1) + q * C1 + co) * 8 + ci;
}
inline uint64_t w1q_bytes(int C1) { return 36ull * 4 * C1 * 8 * 2; }

inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// ResNet-8 weight-gradient splits (every wgrad kernel, the merged SGD reduce and the slot layout follow
// this): layer l's reduction over a batch of `rows` images is cut into r8_split_cap(l, rows) splits of
// whole images.  32x32 layers (0-2): ceil(rows / 2) splits of 2 images (2048 pixels).  16x16 / 8x8
// layers (3-6): S = max(ceil(rows hw / 2048), min(4, ceil(rows / 2))) splits, split s holding images
// [s rows / S, (s + 1) rows / S): at most 2048 pixels, and at least ~4 splits so the light lock-step
// tail's few small-batch clients still spread over many CTAs.  S never decreases with rows, so a slot
// sized for its capacity B (r8_wsp_off) holds every batch's partials, and a full batch touches all of
// them (the observed high-water mark equals the layout, reading R2).  No cohort dependence.
#if defined(__CUDACC__)
__host__ __device__
#endif
inline int r8_split_cap(int layer, int rows) {
  if (layer < 3) return (rows + 1) / 2;
  const int hw = layer < 5 ? 256 : 64, full = (rows * hw + kWgradChunkPx - 1) / kWgradChunkPx;
  const int half = (rows + 1) / 2, floor4 = half < 4 ? half : 4;
  return full > floor4 ? full : floor4;
}
#if defined(__CUDACC__)
__host__ __device__
#endif
inline int r8_split_image(int layer, int rows, int s) {  // first image of split s (s = S: rows)
  return layer < 3 ? (2 * s < rows ? 2 * s : rows) : (int)((int64_t)s * rows / r8_split_cap(layer, rows));
}

// ResNet-8 weight-gradient partials: one region per conv layer (all seven layers' partials are kept
// until the step's single merged SGD reduce), region l = [r8_split_cap(l, B)][cout_l][9 cin_l + 1] fp32
// rows padded to 4 floats.  Float offset of region l (l = 7: the total) for a slot of batch B.
#if defined(__CUDACC__)
__host__ __device__
#endif
inline int64_t r8_wsp_off(int layer, int B) {
  const int co[7] = {16, 16, 16, 32, 32, 64, 64}, ci[7] = {3, 16, 16, 16, 32, 32, 64};
  int64_t off = 0;
  for (int j = 0; j < layer; ++j) off += (int64_t)r8_split_cap(j, B) * co[j] * ((9 * ci[j] + 1 + 3) / 4 * 4);
  return off;
}

}  // namespace protea
