// layout.cpp — model table, FLOP count and the per-client slot layout.
//
// Models (reading R11): MLP 784-64-10; CNN-w (McMahan-style,
// channels 32w/64w/512w); ResNet-8 (6n+2, n=1, option-A shortcut, no BN).
// FLOPs: PAPER.md Table 1 CUDA_time needs a work measure; f = 2 x MACs of
// fwd + wgrad + dgrad without the first layer's dgrad.
#include <algorithm>
#include <cstring>

#include "common.h"

namespace protea {

static Layer conv(int k, int stride, int pad, int cin, int cout, int hin, int win) {
  Layer l{};
  l.kind = 0;
  l.k = k;
  l.stride = stride;
  l.pad = pad;
  l.cin = cin;
  l.cout = cout;
  l.hin = hin;
  l.win = win;
  l.hout = (hin + 2 * pad - k) / stride + 1;
  l.wout = (win + 2 * pad - k) / stride + 1;
  return l;
}

static Layer gnorm(int c) {
  Layer l{};
  l.kind = 2;
  l.cin = c;
  l.cout = c;
  return l;
}

static Layer fc(int in, int out) {
  Layer l{};
  l.kind = 1;
  l.cin = in;
  l.cout = out;
  return l;
}

bool make_model(const protea_model_desc& d, ModelDims* out, std::string* err) {
  ModelDims m;
  m.arch = d.arch;
  m.width_q = d.width_q;
  m.classes = d.classes;
  m.H = d.H;
  m.W = d.W;
  m.C = d.C;
  if (d.classes < 2 || d.classes > 64) {
    *err = "model: classes must be in [2, 64]";
    return false;
  }
  switch (d.arch) {
    case PROTEA_MODEL_MLP:
      if (d.width_q != 4 || d.H * d.W * d.C != 784) {
        *err = "model: MLP needs width_q == 4 and a 784-pixel input (28x28x1)";
        return false;
      }
      m.layers = {fc(784, 64), fc(64, d.classes)};
      break;
    case PROTEA_MODEL_CNN:
      // CIFAR-shaped 32x32x3 (tcgen05 kernels in bf16 mode) or the FEMNIST-shaped 28x28x1 of the paper's
      // LEAF experiment (SIMT kernels in both modes)
      if (!(d.width_q == 1 || d.width_q == 2 || d.width_q == 4) ||
          !((d.H == 32 && d.W == 32 && d.C == 3) || (d.H == 28 && d.W == 28 && d.C == 1))) {
        *err = "model: CNN needs width_q in {1,2,4} and a 32x32x3 or 28x28x1 input";
        return false;
      }
      m.c1 = 8 * d.width_q;
      m.c2 = 16 * d.width_q;
      m.f = 128 * d.width_q;
      m.layers = {conv(5, 1, 2, d.C, m.c1, d.H, d.W), conv(5, 1, 2, m.c1, m.c2, d.H / 2, d.W / 2),
                  fc(d.H / 4 * (d.W / 4) * m.c2, m.f), fc(m.f, d.classes)};
      break;
    case PROTEA_MODEL_RESNET8:
      if (d.width_q != 4 || d.H != 32 || d.W != 32 || d.C != 3) {
        *err = "model: RESNET8 needs width_q == 4 and a 32x32x3 input";
        return false;
      }
      m.layers = {conv(3, 1, 1, 3, 16, 32, 32),  conv(3, 1, 1, 16, 16, 32, 32), conv(3, 1, 1, 16, 16, 32, 32),
                  conv(3, 2, 1, 16, 32, 32, 32), conv(3, 1, 1, 32, 32, 16, 16), conv(3, 2, 1, 32, 64, 16, 16),
                  conv(3, 1, 1, 64, 64, 8, 8),   fc(64, d.classes)};
      break;
    case PROTEA_MODEL_RESNET18: {  // conv (bias), GroupNorm, ReLU; 8 basic blocks, option-A shortcuts (R26)
      if (d.width_q != 4 || d.H != 32 || d.W != 32 || d.C != 3) {
        *err = "model: RESNET18 needs width_q == 4 and a 32x32x3 input";
        return false;
      }
      m.layers = {conv(3, 1, 1, 3, 64, 32, 32), gnorm(64)};
      int cin = 64, hw = 32;
      for (int st = 0; st < 4; ++st) {
        const int c = 64 << st;
        for (int b = 0; b < 2; ++b) {
          const int s = (st > 0 && b == 0) ? 2 : 1;
          m.layers.push_back(conv(3, s, 1, cin, c, hw, hw));
          m.layers.push_back(gnorm(c));
          hw /= s;
          m.layers.push_back(conv(3, 1, 1, c, c, hw, hw));
          m.layers.push_back(gnorm(c));
          cin = c;
        }
      }
      m.layers.push_back(fc(512, d.classes));
      break;
    }
    default:
      *err = "model: unknown arch " + std::to_string(d.arch);
      return false;
  }
  int64_t off = 0;
  for (auto& l : m.layers) {
    l.off_w = off;
    off += (int64_t)l.cout * l.K();
    l.off_b = off;
    off += l.cout;
  }
  m.P = off;
  *out = m;
  return true;
}

uint64_t flops_per_sample(const ModelDims& m) {
  uint64_t fwd = 0, dgrad = 0;
  for (size_t i = 0; i < m.layers.size(); ++i) {
    const Layer& l = m.layers[i];
    if (l.kind == 2) continue;  // GroupNorm: no multiply-accumulates (SURVEY §8(c).3 counts MACs)
    uint64_t macs = l.kind == 0 ? (uint64_t)l.hout * l.wout * l.cout * l.K() : (uint64_t)l.cin * l.cout;
    fwd += macs;
    if (i > 0) dgrad += macs;
  }
  return 2 * (2 * fwd + dgrad);
}

static int splits_for(const Layer& l, int rows) {
  return (int)ceil_div((uint64_t)rows * l.hout * l.wout, kWgradChunkPx);
}

int cnn_conv1_splits(int rows) { return (int)ceil_div((uint64_t)rows * 1024, kWgradChunkPx); }
int cnn_conv2_splits(int rows) { return (int)ceil_div((uint64_t)rows * 256, kWgradChunkPx); }

SlotLayout slot_layout(const ModelDims& m, int b, int64_t n, int epochs, int e) {
  SlotLayout s;
  std::memset(&s, 0, sizeof(s));
  auto put = [&](Buf id, uint64_t bytes) {
    s.used[id] = true;
    s.size[id] = bytes;
  };
  put(B_PARAMS, 4 * (uint64_t)m.P);
  put(B_PERM, 4 * (uint64_t)epochs * n);
  put(B_STATS, 64);
  if (e == 2 && m.arch != PROTEA_MODEL_RESNET18) put(B_WSH, 2 * (uint64_t)m.P);  // bf16 shadow (tensor-core operands)
  // a batch holds min(B, n) rows (the last partial batch is kept): per-row buffers
  // are sized for that many rows (a client with n < B never touches more; observed, tools/hwm_probe.py)
  const uint64_t B = (uint64_t)std::min<int64_t>(b, n);
  if (m.arch == PROTEA_MODEL_MLP) {
    put(B_H1, B * 64 * e);
    put(B_DZ1, B * 64 * e);
  } else if (m.arch == PROTEA_MODEL_CNN) {
    const uint64_t HW = (uint64_t)m.H * m.W, HW2 = HW / 4, HW4 = HW / 16;  // conv1 / conv2 maps, pool-2 output
    put(B_A1, B * HW2 * m.c1 * e);
    put(B_I1, B * HW2 * m.c1);
    put(B_A2, B * HW4 * m.c2 * e);
    put(B_I2, B * HW4 * m.c2);
    put(B_H, B * m.f * e);
    put(B_DH, B * m.f * e);
    put(B_DZ2, B * HW2 * m.c2 * e);
    put(B_DZC1, B * HW * m.c1 * e);
    if (e == 2 && m.H == 32) {  // tcgen05 kernels only
      put(B_XS, B * 36 * 36 * 8 * 2);  // bf16 input staged for the tensor cores: 2-px zero border, ci padded to 8
      put(B_W1P, w1q_bytes(m.c1));     // conv1 pool-quad weight shadow (common.h w1q_index)
    }
  } else if (m.arch == PROTEA_MODEL_RESNET18) {
    int l = 0;
    for (const Layer& x : m.layers)
      if (x.kind == 0) {
        put((Buf)(B_G_Z0 + l), B * x.hout * x.wout * x.cout * e);
        put((Buf)(B_G_Y0 + l), B * x.hout * x.wout * x.cout * e);
        ++l;
      }
    put(B_G_ST, B * kG_Layers * kGroups * 2 * 4);
    put(B_G_X, B * 32 * 32 * 64 * e);
    put(B_G_YG, B * 32 * 32 * 64 * e);
    put(B_G_ZG, B * 32 * 32 * 64 * e);
    put(B_G_GNP, B * 2 * 512 * 4);
  } else {
    put(B_R_A0, B * 1024 * 16 * e);
    put(B_R_R1, B * 1024 * 16 * e);
    put(B_R_O1, B * 1024 * 16 * e);
    put(B_R_R2, B * 256 * 32 * e);
    put(B_R_O2, B * 256 * 32 * e);
    put(B_R_R3, B * 64 * 64 * e);
    put(B_R_O3, B * 64 * 64 * e);
    put(B_R_DGAP, B * 64 * 4);  // (the pooled features stay in the head kernel: no gap buffer)
    put(B_R_G0, B * 1024 * 16 * e);
    put(B_R_G1, B * 1024 * 16 * e);
    put(B_R_G2, B * 1024 * 16 * e);
    if (e == 2) put(B_R_W0P, 16 * 9 * 8 * 2);  // conv0 weight shadow padded to 8 input channels
    if (e == 2) put(B_R_XS, B * 1024 * 8 * 2);  // conv0 input staged for the tensor cores
  }
  // conv weight-gradient split partials: cout rows of K+1 fp32 (K weights + the bias column) per split
  uint64_t wsp = 0;
  const int rows = (int)B;
  if (m.arch == PROTEA_MODEL_RESNET18) {
    for (const Layer& l : m.layers)  // one region reused layer by layer (reduced right after each wgrad)
      if (l.kind == 0) wsp = std::max<uint64_t>(wsp, 4ull * splits_for(l, rows) * l.cout * (l.K() + 1));
  } else if (m.arch == PROTEA_MODEL_RESNET8) {
    // a region per layer (all kept until the step's merged SGD reduce), regions placed at row pitch
    // ceil4(K+1) (r8_wsp_off); the last layer's rows are written at pitch K+1, so its last row ends the slot
    wsp = 4ull * ((uint64_t)r8_wsp_off(6, rows) + (uint64_t)r8_split_cap(6, rows) * 64 * (9 * 64 + 1));
  } else if (m.arch == PROTEA_MODEL_CNN && e == 2 && m.width_q == 4 && m.H == 32) {
    // width 1, bf16: conv1's partials live in dz2 (k_conv1_wgrad_q); conv2 writes partials (row pitch
    // ceil4(K+1) = 804) only when a client's rows need more than one split, else it updates from TMEM
    const int s2 = splits_for(m.layers[1], rows);
    if (s2 > 1) wsp = 4ull * s2 * m.c2 * ((m.layers[1].K() + 1 + 3) / 4 * 4);
  } else {
    for (const Layer& l : m.layers)  // one region reused layer by layer (max), rows at pitch K+1
      if (l.kind == 0) wsp = std::max<uint64_t>(wsp, 4ull * splits_for(l, rows) * l.cout * (l.K() + 1));
  }
  if (wsp) put(m.arch == PROTEA_MODEL_RESNET8 ? B_R_WSP : m.arch == PROTEA_MODEL_RESNET18 ? B_G_WSP : B_WSP, wsp);
  // slot order = enum order except that the wgrad partials come last (oracle order)
  uint64_t off = 0;
  for (int i = 0; i < B_COUNT; ++i) {
    if (!s.used[i] || i == B_WSP || i == B_R_WSP || i == B_G_WSP) continue;
    s.off[i] = off;
    off += align256(s.size[i]);
  }
  for (int i : {B_WSP, B_R_WSP, B_G_WSP})
    if (s.used[i]) {
      s.off[i] = off;
      off += align256(s.size[i]);
    }
  s.total = off;
  return s;
}

uint64_t client_hwm(const ModelDims& m, int batch, int64_t n, int epochs, int e) {
  const int64_t b = std::min<int64_t>(batch, n);
  if (b <= kMicroRows) return slot_layout(m, batch, n, epochs, e).total;
  uint64_t tot = 0;
  for (int64_t r0 = 0; r0 < b; r0 += kMicroRows)
    tot += slot_layout(m, (int)std::min<int64_t>(kMicroRows, b - r0), n, epochs, e).total;
  return tot + align256(4 * (uint64_t)m.P);  // merge weights
}

}  // namespace protea
