// engine.cu — the virtual-client engine and the C ABI (include/protea.h).
//
// PAPER.md §3.2: the VCE runs "as many clients concurrently as the
// available system resources can hold" and spawns the next one when a client
// finishes.  Here the "resource" is a byte range of this GPU's arena (the slot
// of protea_plan) and concurrency is realised as LOCK-STEP ITERATIONS: in
// iteration t every admitted client (admit <= t < release) advances one local
// SGD step, and every layer-op of that step is ONE grouped kernel launch over
// all active clients (kernels_simt.cuh).  Clients are admitted / released at
// the iterations the plan fixed; on release the client's FedAvg term
// n_k (w_k - w_g) is added to the group's fp64 accumulator, and after
// the last iteration the ranks sum their accumulators (NCCL, the only
// cross-GPU exchange) and every rank writes w' = w_g + acc / N.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges visible to nsys / ncu --nvtx when a tool is attached

#include <array>
#include <tuple>
#include <type_traits>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "common.h"
#include "device.cuh"
#include "kernels_misc.cuh"
#include "kernels_simt.cuh"
#include "kernels_tc.cuh"
#include "kernels_conv.cuh"
#include "kernels_resnet.cuh"
#include "kernels_resnet_tc.cuh"
#include "kernels_resnet_halo.cuh"
#include "kernels_resnet18.cuh"

namespace protea {
// NVTX range for the enclosing scope (round phases and lock-step iterations; SURVEY §5 tracing)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

static std::mutex g_err_mu;
static std::string g_err;
void set_global_error(const std::string& msg) {
  std::lock_guard<std::mutex> lk(g_err_mu);
  g_err = msg;
}

struct Group {
  ModelDims m;
  int64_t offset = 0;  // in the concatenated global vector
};

struct ShardDev {
  int64_t n = 0;
  uint8_t* x = nullptr;
  int32_t* y = nullptr;
  int32_t ymin = 0, ymax = 0;  // label range (scanned at registration; run_round checks it against the model)
};

template <typename T>
struct DevArray {
  T* p = nullptr;
  size_t cap = 0;
  cudaError_t reserve(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T));
    if (e == cudaSuccess) cap = n;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

}  // namespace protea

using namespace protea;

struct protea_ctx {
  int device = 0, rank = 0, world = 1, precision = PROTEA_PREC_FP32;
  cudaStream_t stream = nullptr;
  uint8_t* arena = nullptr;
  uint64_t arena_bytes = 0;
  std::vector<Group> groups;
  std::map<int64_t, ShardDev> shards;
  std::map<int64_t, ShardDev> val_shards;  // validation splits, protea_register_val_shards
  bool eval_mode = false;                  // execute(): forward + k_eval_head only (evaluate round)
  ncclComm_t comm = nullptr;
  std::string err;
  DevArray<float> gin, gout;
  DevArray<double> acc;
  DevArray<double> gath;     // K7: all-gathered per-rank partials [world][P + groups]
  DevArray<uint64_t> flag;   // plan hash / error flags exchanged before and after a round
  DevArray<uint64_t> regions;          // observed HWMs: (offset, bytes) per slot / guard region
  DevArray<unsigned long long> hwm;    // observed HWMs: 1 + highest touched byte per region
  DevArray<ClientRec> recs;
  DevArray<int32_t> tab;
  // protea_evaluate workspace (kept apart from the round's tables)
  DevArray<ClientRec> ev_recs;
  DevArray<int32_t> ev_tab;
  DevArray<uint8_t> ev_ws;
  DevArray<double> ev_loss;
  DevArray<uint32_t> ev_ok;
  DevArray<const float*> ptrs;
  DevArray<double> wts;
  DevArray<int32_t> wq;  // protea_heterofl_aggregate: client widths
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  uint64_t launches = 0;
  // side stream: fc1 wgrad (HBM-bound weight RMW) overlaps the conv backward chain (L2 / tensor bound)
  cudaStream_t side = nullptr;  // lowest priority: the deferred fc1 wgrad
  cudaStream_t hi = nullptr;    // highest priority: the lock-step chain of execute()
  cudaStream_t cur = nullptr;  // stream the launch helpers currently issue to
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  std::vector<cudaEvent_t> gjoin;  // per model group: end of its deferred fc1 wgrad
  // per model group: its own high-priority lock-step stream (the groups' chains are independent within
  // a round: different clients, weights and FedAvg accumulators), with an event to join it
  std::vector<cudaStream_t> gstream;
  std::vector<cudaEvent_t> gdone;
  std::vector<char> gpending;      // per model group: a deferred fc1 wgrad not yet joined
  bool overlap_now = false;        // current iteration defers fc1 wgrad (light iteration)
  // programmatic dependent launch on the lock-step stream (PROTEA_PDL=0 turns it off): the next kernel's
  // prologue (barriers, TMEM, its first client's weights) overlaps the previous kernel's drain.  Round 1
  // measured it slower (config 2: 70.2 -> 71.5 ms); with round 2's kernels it is faster: config 2
  // 63.5 -> 62.0 ms, config 5 44.1 -> 42.5 ms (tools/env_sweep.sh)
  bool pdl = true;
  int f1w_side_smem = 0;
  bool defer_c2r = true;
  bool single_chain = true;
  // ResNet-8 bf16 backward: layer i's wgrad on its own stream beside layer i's dgrad (PROTEA_R8_OVERLAP)
  bool r8_overlap = true;
  int64_t r8_overlap_rows = 1024;  // ... in iterations of at most this many rows (PROTEA_R8_OVERLAP_ROWS)
  int64_t rows_now = 0;            // rows of the current lock-step iteration (all groups)
  cudaStream_t wstream = nullptr;
  cudaEvent_t r8ev[16] = {};  // this round's lock-step chain is one stream (one group, one lane)  // width-1 conv2 wgrad split reduce on the side stream (PROTEA_DEFER_C2R=0: in-kernel)  // deferred fc1 wgrad: dynamic smem floor (PROTEA_F1W_SIDE_SMEM), limits its CTAs per SM
  int lanes = 1;     // lock-step lanes per model group (PROTEA_LANES): independent chains on own streams
  int spin_cap = 148;  // CTAs of a kernel whose CTAs spin-wait on each other (the width-1 CNN wgrad split
                       // reduces): g_num_sms / lanes, so concurrent lanes' instances are all co-resident
  int64_t overlap_rows = 300;  // defer when the iteration has at most this many rows (PROTEA_OVERLAP_ROWS); round 2 sweep: 0 / 300 / 640 / 1000 / 1500 rows -> 57.50 / 57.52 / 58.36 / 58.45 / 58.89 ms
  // per-op-class accounting of the current round (protea_round_stats)
  uint32_t time_ops = 0;
  bool serialize = false;  // this round: no side-stream deferral (protea_round_opts.serialize)
  std::vector<cudaEvent_t> evpool;
  size_t evused = 0;
  std::vector<int> ev_op;
  std::vector<std::pair<uint64_t, uint64_t>> ev_work;  // (flops, bytes) of each timed launch
  const uint64_t* cur_fl = nullptr;                  // per-op work of the launch being issued (Launch::fl/by)
  const uint64_t* cur_by = nullptr;
  uint64_t op_launches[PROTEA_N_OPC] = {}, op_flops[PROTEA_N_OPC] = {}, op_bytes[PROTEA_N_OPC] = {};
  double loss_host = 0.0;
  // partial-round state (protea_round_partial / protea_round_finalize)
  bool have_partial = false;
  std::vector<int64_t> last_Ngroup;
  // TMA tensor maps per (client, slot offset, batch, group), reused across rounds
  std::map<std::tuple<uint64_t, int, int, int64_t, int>, std::array<CUtensorMap, kTmapSlots>> tmap_cache;  // (offset, B, E, n, group): everything the slot layout depends on
  DevArray<CUtensorMap> tmaps;
  DevArray<uint64_t> smns;  // K9 per-client SM-time counters of the current round
};

namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool tmap_encode(CUtensorMap* m, const void* addr, int rank, const uint64_t* dims, const uint64_t* strides,
                 const uint32_t* box, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE) {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&g_encode, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !g_encode)
      return false;
  }
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(addr), (const cuuint64_t*)dims,
                  (const cuuint64_t*)strides, (const cuuint32_t*)box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The TMA tensor maps of one bf16-mode CNN client (see TmapId in kernels_tc.cuh).
bool build_cnn_tmaps(const ModelDims& m, const ClientRec& r, int B, CUtensorMap* out) {
  const uint64_t C1 = m.c1, C2 = m.c2, F = m.f, K1 = 64 * C2, Bk = B, R = (B + 15) & ~15;
  const uint8_t* wsh = (const uint8_t*)r.buf[B_WSH];
  const void* w2 = wsh + 2 * m.layers[1].off_w;
  const void* w3 = (const uint8_t*)r.buf[B_PARAMS] + 4 * m.layers[2].off_w;  // fc1 W: hi split plane
  bool ok = true;
  {
    const uint64_t d[4] = {C1, 16, 16, Bk}, st[3] = {C1 * 2, 32 * C1, 512 * C1};
    const uint32_t b8[4] = {8, 16, 8, 1}, b4[4] = {8, 16, 4, 1}, b12[4] = {8, 16, 12, 1}, w12[4] = {32, 16, 12, 1};
    ok &= tmap_encode(&out[TM_A1], r.buf[B_A1], 4, d, st, b8);
    ok &= tmap_encode(&out[TM_A1W], r.buf[B_A1], 4, d, st, b4);
    if (C1 >= 32)  // halo copies: 32-channel boxes, 64-byte swizzle (HaloGeom::SW64)
      ok &= tmap_encode(&out[TM_A1H], r.buf[B_A1], 4, d, st, w12, CU_TENSOR_MAP_SWIZZLE_64B);
    else
      ok &= tmap_encode(&out[TM_A1H], r.buf[B_A1], 4, d, st, b12);
  }
  {
    const uint64_t d[4] = {C2, 16, 16, Bk}, st[3] = {C2 * 2, 32 * C2, 512 * C2};
    const uint32_t b8[4] = {8, 16, 8, 1}, b4[4] = {8, 16, 4, 1}, b12[4] = {8, 16, 12, 1}, w12[4] = {32, 16, 12, 1};
    ok &= tmap_encode(&out[TM_DZ2W], r.buf[B_DZ2], 4, d, st, b4);
    if (C2 >= 32)
      ok &= tmap_encode(&out[TM_DZ2H], r.buf[B_DZ2], 4, d, st, w12, CU_TENSOR_MAP_SWIZZLE_64B);
    else
      ok &= tmap_encode(&out[TM_DZ2H], r.buf[B_DZ2], 4, d, st, b12);
  }
  {
    const uint64_t d[2] = {25 * C1, C2}, st[1] = {50 * C1};
    const uint32_t bx[2] = {8, (uint32_t)C2};
    ok &= tmap_encode(&out[TM_W2F], w2, 2, d, st, bx);
  }
  {
    const uint64_t d[3] = {C1, 25, C2}, st[2] = {2 * C1, 50 * C1};
    const uint32_t bx[3] = {8, 1, (uint32_t)C2};
    ok &= tmap_encode(&out[TM_W2D], w2, 3, d, st, bx);
  }
  {  // fc1 W upper halves: [F][K1 / 128][128] bf16, 128-blocks 512 B apart (the lower halves in between)
    const uint64_t d[3] = {128, K1 / 128, F}, st[2] = {512, 4 * K1};
    const uint32_t bk[3] = {64, 1, 128}, bm[3] = {64, 1, 64};
    ok &= tmap_encode(&out[TM_W3K], w3, 3, d, st, bk, CU_TENSOR_MAP_SWIZZLE_128B);
    ok &= tmap_encode(&out[TM_W3M], w3, 3, d, st, bm, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  {
    const uint64_t d[2] = {K1, Bk}, st[1] = {2 * K1};
    const uint32_t bx[2] = {64, (uint32_t)R};
    ok &= tmap_encode(&out[TM_A2], r.buf[B_A2], 2, d, st, bx, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  if (C1 == 32 && C2 == 64) {  // width 1: single-halo conv2 kernels (kernels_conv.cuh)
    const uint64_t d1[4] = {C1, 16, 16, Bk}, s1[3] = {C1 * 2, 32 * C1, 512 * C1};
    const uint64_t d2[4] = {C2, 16, 16, Bk}, s2[3] = {C2 * 2, 32 * C2, 512 * C2};
    const uint32_t bq1[4] = {32, 12, 20, 1}, bq2[4] = {64, 8, 16, 1};
    ok &= tmap_encode(&out[TM_A1Q], r.buf[B_A1], 4, d1, s1, bq1, CU_TENSOR_MAP_SWIZZLE_64B);
    ok &= tmap_encode(&out[TM_DZ2Q], r.buf[B_DZ2], 4, d2, s2, bq2, CU_TENSOR_MAP_SWIZZLE_128B);
    ok &= tmap_encode(&out[TM_DZ2Q1], r.buf[B_DZ2], 4, d2, s2, bq1, CU_TENSOR_MAP_SWIZZLE_64B);
    const uint64_t dwf[2] = {25 * C1, C2}, swf[1] = {50 * C1};
    const uint32_t bwf[2] = {64, 64};
    ok &= tmap_encode(&out[TM_W2FS], w2, 2, dwf, swf, bwf, CU_TENSOR_MAP_SWIZZLE_128B);
    const uint64_t dwd[3] = {C1, 25, C2}, swd[2] = {2 * C1, 50 * C1};
    const uint32_t bwd[3] = {32, 1, 64};
    ok &= tmap_encode(&out[TM_W2DS], w2, 3, dwd, swd, bwd, CU_TENSOR_MAP_SWIZZLE_64B);
  }
  if (r.buf[B_XS]) {  // staged input xs[B][36 Y][2 par][18 X' x 8 ch] (k_stage_x): pixel runs as the inner dim
    const uint64_t dx[4] = {144, 2, 36, Bk}, sx[3] = {288, 576, 36 * 576};
    const uint32_t bh[4] = {80, 2, 36, 1}, bw[4] = {64, 1, 36, 1};
    ok &= tmap_encode(&out[TM_XSH], r.buf[B_XS], 4, dx, sx, bh);
    ok &= tmap_encode(&out[TM_XSW], r.buf[B_XS], 4, dx, sx, bw);
  }
  if (r.buf[B_XS] && C1 == 32) {  // pool-quad conv1 gradient g1[B][16][16][4 q][C1] (k_conv1_wgrad_q)
    const uint64_t d[4] = {4 * C1, 16, 16, Bk}, st[3] = {8 * C1, 128 * C1, 2048 * C1};
    const uint32_t bx[4] = {64, 8, 16, 1};
    ok &= tmap_encode(&out[TM_G], r.buf[B_DZC1], 4, d, st, bx, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  {
    const uint64_t d[2] = {F, Bk}, st[1] = {2 * F};
    const uint32_t bx[2] = {64, (uint32_t)R};
    ok &= tmap_encode(&out[TM_DH], r.buf[B_DH], 2, d, st, bx, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  return ok;
}

// ResNet-8 layers run by the halo kernels (kernels_resnet_halo.cuh): stride 1, C -> C, with C = 16 / 32 / 64
// at 32x32 / 16x16 / 8x8.  PROTEA_R8_HALO = bit mask 1 fwd, 2 dgrad, 4 wgrad, 8 conv0 too (default 15; a
// cleared bit runs that pass on the gathered kernels of kernels_resnet_tc.cuh).
int g_r8_halo = 15;
enum { R8H_FWD = 1, R8H_DGRAD = 2, R8H_WGRAD = 4 };
int r8_halo_c(const Layer& l, int pass) {
  if (!(g_r8_halo & pass) || l.kind != 0 || l.k != 3 || l.stride != 1 || l.cin != l.cout) return 0;
  const int c = l.cin;
  return ((c == 16 && l.hin == 32) || (c == 32 && l.hin == 16) || (c == 64 && l.hin == 8)) && l.win == l.hin ? c : 0;
}
int r8_halo_tiles(int c) { return c == 16 ? 8 : c == 32 ? 2 : 1; }
// conv0 (3 -> 16 at 32x32, on the staged input) on RHalo0 / RWgHalo0
bool r8_halo0(const Layer& l, int pass) {
  return (g_r8_halo & 8) && (g_r8_halo & pass) && l.kind == 0 && l.k == 3 && l.stride == 1 && l.cin == 3 &&
         l.cout == 16 && l.hin == 32 && l.win == 32;
}
// stride-2 fwd halo (RHaloS2): 16 -> 32 at 32x32 and 32 -> 64 at 16x16; returns Cin
int r8_halo_s2(const Layer& l, int pass = R8H_FWD) {
  if (!(g_r8_halo & pass) || l.kind != 0 || l.k != 3 || l.stride != 2 || l.cout != 2 * l.cin) return 0;
  return ((l.cin == 16 && l.hin == 32) || (l.cin == 32 && l.hin == 16)) && l.win == l.hin ? l.cin : 0;
}

// The TMA tensor maps of one bf16-mode ResNet-8 client (RTmapId): the halo boxes (C, 10, 18, 1) of the
// stride-1 layers' inputs (fwd) and output gradients (dgrad), and their weight taps (C, 1, C).
bool build_r8_tmaps(const ModelDims& m, const ClientRec& r, int B, CUtensorMap* out) {
  static const int lay[4] = {1, 2, 4, 6};
  static const int in_buf[4] = {B_R_A0, B_R_R1, B_R_R2, B_R_R3};
  static const int dout_buf[4] = {B_R_G2, B_R_G1, B_R_G2, B_R_G0};  // launch_step_resnet's gradient rotation
  bool ok = true;
  for (int k = 0; k < 4; ++k) {
    const Layer& l = m.layers[lay[k]];
    const uint64_t C = l.cin, H = l.hin;
    if (!r8_halo_c(l, 7)) continue;
    const CUtensorMapSwizzle sw = C == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : C == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                                          : CU_TENSOR_MAP_SWIZZLE_128B;
    const uint64_t d[4] = {C, H, H, (uint64_t)B}, st[3] = {2 * C, 2 * C * H, 2 * C * H * H};
    const uint32_t box[4] = {(uint32_t)C, 10, 18, 1};
    ok &= tmap_encode(&out[RTM_IN1 + k], r.buf[in_buf[k]], 4, d, st, box, sw);
    ok &= tmap_encode(&out[RTM_DO1 + k], r.buf[dout_buf[k]], 4, d, st, box, sw);
    const uint32_t tbox[4] = {(uint32_t)C, 8, 18, 1};  // (RWgHalo: one dout row above and below the tile)
    ok &= tmap_encode(&out[RTM_WD1 + k], r.buf[dout_buf[k]], 4, d, st, tbox, sw);
    const uint64_t dw[3] = {C, 9, C}, sw_[2] = {2 * C, 18 * C};
    const uint32_t bw[3] = {(uint32_t)C, 1, (uint32_t)C};
    ok &= tmap_encode(&out[RTM_W1 + k], (const uint8_t*)r.buf[B_WSH] + 2 * l.off_w, 3, dw, sw_, bw, sw);
  }
  if (r8_halo0(m.layers[0], R8H_FWD | R8H_WGRAD)) {  // conv0: staged input rows, padded weight taps, dz0 tiles
    const uint64_t d[3] = {256, 32, (uint64_t)B}, st[2] = {512, 16384};
    const uint32_t box[3] = {80, 19, 1};  // (RHalo0::HBYTES)
    ok &= tmap_encode(&out[RTM_IN0], r.buf[B_R_XS], 3, d, st, box);
    const uint64_t dw[3] = {8, 9, 16}, sw_[2] = {16, 144};
    const uint32_t bw[3] = {8, 1, 16};
    ok &= tmap_encode(&out[RTM_W0], r.buf[B_R_W0P], 3, dw, sw_, bw);
    const uint64_t dd[4] = {16, 32, 32, (uint64_t)B}, sd[3] = {32, 1024, 32768};
    const uint32_t bt[4] = {16, 8, 18, 1};
    ok &= tmap_encode(&out[RTM_WD0], r.buf[B_R_G0], 4, dd, sd, bt, CU_TENSOR_MAP_SWIZZLE_32B);
  }
  static const int lay2[2] = {3, 5}, in2[2] = {B_R_O1, B_R_O2};
  for (int k = 0; k < 2; ++k) {  // stride-2 fwd: the input as pixel pairs [B][H][W/2][2 Cin]
    const Layer& l = m.layers[lay2[k]];
    if (!r8_halo_s2(l, 7)) continue;
    const uint64_t C = l.cin, H = l.hin, Co = l.cout;
    const CUtensorMapSwizzle sw = C == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B;
    const uint64_t d[4] = {2 * C, H / 2, H, (uint64_t)B}, st[3] = {4 * C, 2 * C * H, 2 * C * H * H};
    const uint32_t box[4] = {(uint32_t)C, 9, 33, 1};
    ok &= tmap_encode(&out[RTM_IN3 + k], r.buf[in2[k]], 4, d, st, box, sw);
    const uint64_t dw[3] = {C, 9, Co}, sw_[2] = {2 * C, 18 * C};
    const uint32_t bw[3] = {(uint32_t)C, 1, (uint32_t)Co};
    ok &= tmap_encode(&out[RTM_W3 + k], (const uint8_t*)r.buf[B_WSH] + 2 * l.off_w, 3, dw, sw_, bw, sw);
    const uint64_t Ho = H / 2, dd[4] = {Co, Ho, Ho, (uint64_t)B}, sd[3] = {2 * Co, 2 * Co * Ho, 2 * Co * Ho * Ho};
    const uint32_t bd[4] = {(uint32_t)Co, 9, 17, 1};
    ok &= tmap_encode(&out[RTM_DO3 + k], r.buf[k == 0 ? B_R_G0 : B_R_G1], 4, dd, sd, bd,
                      Co == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B);
    const uint32_t bt[4] = {(uint32_t)Co, 8, 16, 1};
    ok &= tmap_encode(&out[RTM_WD3 + k], r.buf[k == 0 ? B_R_G0 : B_R_G1], 4, dd, sd, bt,
                      Co == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B);
  }
  return ok;
}
}  // namespace

namespace {
// Bracket one launch of op class `op` with CUDA events if requested.
int op_begin(protea_ctx* ctx, int op, int raw = -1) {  // op: stats class; raw: launch op id (work lookup)
  if (op < 0 || op >= PROTEA_N_OPC) op = PROTEA_N_OPC - 1;  // (defensive: never index past the stats arrays)
  ctx->op_launches[op]++;
  ctx->launches++;
  if (!((ctx->time_ops >> op) & 1u)) return -1;
  if (ctx->cur == ctx->side && ctx->side != ctx->stream) return -1;  // concurrent with other kernels: not timed
  while (ctx->evused + 2 > ctx->evpool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    ctx->evpool.push_back(e);
  }
  const int i = (int)ctx->evused;
  ctx->evused += 2;
  ctx->ev_op.push_back(op);
  ctx->ev_work.emplace_back(raw >= 0 && ctx->cur_fl ? ctx->cur_fl[raw] : 0, raw >= 0 && ctx->cur_by ? ctx->cur_by[raw] : 0);
  cudaEventRecord(ctx->evpool[i], ctx->cur);
  return i;
}
void op_end(protea_ctx* ctx, int i) {
  if (i >= 0) cudaEventRecord(ctx->evpool[i + 1], ctx->cur);
}
// Launch on ctx->cur; on the lock-step stream with programmatic stream serialization (PDL) so the kernel's
// CTAs can run their prologue while the preceding kernel drains (kernels call pdl_wait(), device.cuh).
template <typename... KArgs, typename... Args>
void launch_k(protea_ctx* ctx, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->cur;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (ctx->pdl && ctx->cur == ctx->hi) ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, args...);
}
void reset_ops(protea_ctx* ctx, uint32_t time_ops) {
  ctx->time_ops = time_ops;
  ctx->evused = 0;
  ctx->ev_op.clear();
  ctx->ev_work.clear();
  for (int i = 0; i < PROTEA_N_OPC; ++i) ctx->op_launches[i] = ctx->op_flops[i] = ctx->op_bytes[i] = 0;
}
}  // namespace

#define CK(call)                                                                               \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) {                                                                   \
      ctx->err = std::string("CUDA error ") + cudaGetErrorString(e_) + " at " #call;           \
      return PROTEA_ERR_CUDA;                                                                  \
    }                                                                                          \
  } while (0)

static protea_status fail(protea_ctx* ctx, protea_status s, const std::string& m) {
  ctx->err = m;
  return s;
}

// ---------------------------------------------------------------------------
// per-model op tables: tile counts (must mirror the device setup() decode)
// ---------------------------------------------------------------------------
namespace {

constexpr int kMaxBatch = 4096;  // batches above kMicroRows rows run as micro-clients (common.h)

// tile shapes
constexpr int C1F_BM = 64, C1F_BN = 32;
constexpr int C2F_BM = 64, C2F_BN = 64;
constexpr int F1F_BM = 32, F1F_BN = 64;
constexpr int F1D_BM = 32, F1D_BN = 64;
constexpr int F1W_BM = 64, F1W_BN = 64;
constexpr int C2D_BM = 64, C2D_BN = 32;
constexpr int C2W_BM = 64, C2W_BN = 64;
constexpr int C1W_BM = 32, C1W_BN = 64;
constexpr int MF_BM = 16, MF_BN = 64;
constexpr int MW_BM = 64, MW_BN = 64;

enum Op : int {
  OP_C1F = 0, OP_C2F, OP_F1F, OP_HEAD, OP_F1D, OP_F1W, OP_C2D, OP_C2W, OP_C2R, OP_C1W, OP_C1R,
  OP_MF, OP_MHEAD, OP_MW, OP_ADMIT_, OP_FEDAVG_, OP_STAGE,
  // ResNet-8 launch instances (each needs its own prefix table); stats use PROTEA_OPC_R_* classes
  RI_F0 = 32, RI_HEAD = RI_F0 + 7, RI_D1 = RI_HEAD + 1, RI_W0 = RI_D1 + 6, RI_R0 = RI_W0 + 7,
  // ResNet-18 (GroupNorm) launch instances, 17 conv layers each: conv fwd, GroupNorm fwd, head, GroupNorm
  // bwd, GroupNorm reduce, conv dgrad (layer 0 unused), conv wgrad, conv reduce
  GI_F = RI_R0 + 7, GI_N = GI_F + 17, GI_HEAD = GI_N + 17, GI_NB = GI_HEAD + 1, GI_NR = GI_NB + 17,
  GI_D = GI_NR + 17, GI_W = GI_D + 17, GI_R = GI_W + 17, OP_COUNT = GI_R + 17
};
// ResNet-8 SIMT tile shape
constexpr int R_BM = 64, R_BN = 32;
const protea::Layer& rlayer(const ModelDims& m, int i) { return m.layers[i]; }
int rsplits(const Layer& l, int rows) { return cdiv(rows * l.hout * l.wout, kWgradChunkPx); }

// tensor-core tile shapes (bf16 mode): M tile = 128, BN per op, STAGES-deep ring
constexpr int TC_C1F_BN = 32, TC_C1W_BN = 32, TC_C2F_BN = 64, TC_C2D_BN = 32, TC_C2W_BN = 64, TC_F1F_BN = 64, TC_F1D_BN = 64, TC_F1W_BN = 128;
constexpr int TC_STAGES = 4, TC_F1W_STAGES = 1, TC_F1F_STAGES = 8;
// Join a group's deferred fc1 wgrad into the current stream (before anything that writes a2 / dh
// or reads the fc1 weights: the next conv2 fwd, a release, the end of the round).
void join_group(protea_ctx* ctx, int g) {
  if (g < (int)ctx->gpending.size() && ctx->gpending[g]) {
    cudaStreamWaitEvent(ctx->cur, ctx->gjoin[g], 0);
    ctx->gpending[g] = 0;
  }
}

const Layer& gconv(const ModelDims& m, int l) { return m.layers[2 * l]; }  // ResNet-18 conv layer l (0..16)
const Layer& gnorm_of(const ModelDims& m, int l) { return m.layers[2 * l + 1]; }

int tiles(const ModelDims& m, int op, int rows, bool tc) {
  if (op >= GI_F) {  // ResNet-18: SIMT kernels
    if (op == GI_HEAD) return 1;
    if (op < GI_N) {
      const Layer& l = gconv(m, op - GI_F);
      return cdiv(rows * l.hout * l.wout, R_BM) * cdiv(l.cout, R_BN);
    }
    if (op < GI_HEAD || (op >= GI_NB && op < GI_NR)) return rows * kGroups;
    if (op < GI_D) return 1;  // GroupNorm reduce: one CTA per client
    if (op < GI_W) {
      const Layer& l = gconv(m, op - GI_D);
      return cdiv(rows * l.hin * l.win, R_BM) * cdiv(l.cin, R_BN);
    }
    if (op < GI_R) {
      const Layer& l = gconv(m, op - GI_W);
      return rsplits(l, rows) * cdiv(l.cout, R_BM) * cdiv(9 * l.cin + 1, R_BN);
    }
    const Layer& l = gconv(m, op - GI_R);
    return cdiv(l.cout * (9 * l.cin + 1), kReduceBlock);
  }
  if (m.arch == PROTEA_MODEL_CNN && m.H != 32) tc = false;  // FEMNIST-shaped CNN: SIMT kernels
  const int HW = m.H * m.W, HW2 = HW / 4, K1 = HW / 16 * m.c2, KC1 = 25 * m.C + 1;
  if (op >= RI_F0) {
    if (op == RI_HEAD) return 1;
    // bf16 mode: every conv on tcgen05 (kernels_resnet_tc.cuh), 128-row tiles (conv0 on the staged input)
    if (op < RI_HEAD) {
      const Layer& l = m.layers[op - RI_F0];
      if (tc && r8_halo_c(l, R8H_FWD)) return rows * r8_halo_tiles(l.cin);  // halo kernels: 16 x 8 pixel tiles
      if (tc && r8_halo0(l, R8H_FWD)) return rows * 8;
      if (tc && r8_halo_s2(l)) return rows * (l.cin == 16 ? 2 : 1);
      if (tc) return cdiv(rows * l.hout * l.wout, 128);
      return cdiv(rows * l.hout * l.wout, R_BM) * cdiv(l.cout, R_BN);
    }
    if (op < RI_W0) {
      const Layer& l = m.layers[1 + op - RI_D1];
      if (tc && r8_halo_c(l, R8H_DGRAD)) return rows * r8_halo_tiles(l.cin);
      if (tc && r8_halo_s2(l, R8H_DGRAD)) return rows * (l.cin == 16 ? 8 : 4);  // 4 parity classes
      if (tc) return cdiv(rows * l.hin * l.win, 128);
      return cdiv(rows * l.hin * l.win, R_BM) * cdiv(l.cin, R_BN);
    }
    if (op < RI_R0) {
      const Layer& l = m.layers[op - RI_W0];
      const int sp = r8_split_cap(op - RI_W0, rows);  // (common.h: whole-image splits)
      if (tc && (r8_halo_c(l, R8H_WGRAD) || r8_halo_s2(l, R8H_WGRAD) || r8_halo0(l, R8H_WGRAD)))
        return sp;  // halo wgrad: one item per split
      if (tc) return sp * cdiv(9 * (l.cin < 8 ? 8 : l.cin) + 1, 128);
      return sp * cdiv(l.cout, R_BM) * cdiv(9 * l.cin + 1, R_BN);
    }
    const Layer& l = m.layers[op - RI_R0];
    return cdiv(l.cout * (9 * l.cin + 1), kReduceBlock);
  }
  if (tc) switch (op) {
      case OP_STAGE: return cdiv(rows * 1296, kStageThreads);
      case OP_C1F: return rows * 2;  // persistent pool-quad kernel: 2 tiles of 128 pooled pixels per image
      case OP_C1W:  // width 1: persistent pool-quad kernel, one item per split; else 2 M tiles per split
        return m.width_q == 4 ? cdiv(rows, w1q_ips(rows)) : 2 * cdiv(rows * 1024, kWgradChunkPx);
      case OP_C1R: return cdiv(76 * m.c1, kReduceBlock);
      case OP_C2F: return rows * 2;  // halo kernel (width >= 1/2) or TmaConv2Fwd: both 128-pixel tiles
      case OP_F1F: return m.f / 128;
      case OP_F1D: return 64 * m.c2 / 128;
      case OP_F1W: return (64 * m.c2 / 128) * cdiv(m.f, 128);
      case OP_C2D: return rows * 2;
      case OP_C2W:  // width 1: persistent halo kernel, one item per split; else one CTA per (split, M tile)
        return cdiv(rows * 256, kWgradChunkPx) * (m.width_q == 4 ? 1 : cdiv(25 * m.c1 + 1, 128));
      default: break;
    }
  switch (op) {
    case OP_C1F: return cdiv(rows * HW, C1F_BM) * cdiv(m.c1, C1F_BN);
    case OP_C2F: return cdiv(rows * HW2, C2F_BM) * cdiv(m.c2, C2F_BN);
    case OP_F1F: return cdiv(rows, F1F_BM) * cdiv(m.f, F1F_BN);
    case OP_HEAD: return 1;  // k_head_cnn: one CTA per client
    case OP_F1D: return cdiv(rows, F1D_BM) * cdiv(K1, F1D_BN);
    case OP_F1W: return cdiv(m.f, F1W_BM) * cdiv(K1, F1W_BN);
    case OP_C2D: return cdiv(rows * HW2, C2D_BM) * cdiv(m.c1, C2D_BN);
    case OP_C2W: return cdiv(rows * HW2, kWgradChunkPx) * cdiv(m.c2, C2W_BM) * cdiv(25 * m.c1 + 1, C2W_BN);
    case OP_C2R: return cdiv(m.c2 * (25 * m.c1 + 1), kReduceBlock);
    case OP_C1W: return cdiv(rows * HW, kWgradChunkPx) * cdiv(m.c1, C1W_BM) * cdiv(KC1, C1W_BN);
    case OP_C1R: return cdiv(m.c1 * KC1, kReduceBlock);
    case OP_MF: return cdiv(rows, MF_BM) * cdiv(64, MF_BN);
    case OP_MHEAD: return 1;
    case OP_MW: return cdiv(64, MW_BM) * cdiv(784, MW_BN);
  }
  return 0;
}

std::vector<int> ops_of(const ModelDims& m, bool tc) {
  tc = tc && (m.arch != PROTEA_MODEL_CNN || m.H == 32);  // the tcgen05 CNN kernels are 32x32x3-only
  if (m.arch == PROTEA_MODEL_CNN && tc && m.width_q == 4)  // conv1 reduce fused into k_conv1_wgrad_q
    return {OP_STAGE, OP_C1F, OP_C2F, OP_F1F, OP_HEAD, OP_F1D, OP_F1W, OP_C2D, OP_C2W, OP_C1W};
  if (m.arch == PROTEA_MODEL_CNN && tc)
    return {OP_STAGE, OP_C1F, OP_C2F, OP_F1F, OP_HEAD, OP_F1D, OP_F1W, OP_C2D, OP_C2W, OP_C1W, OP_C1R};
  if (m.arch == PROTEA_MODEL_CNN)
    return {OP_C1F, OP_C2F, OP_F1F, OP_HEAD, OP_F1D, OP_F1W, OP_C2D, OP_C2W, OP_C2R, OP_C1W, OP_C1R};
  if (m.arch == PROTEA_MODEL_MLP) return {OP_MF, OP_MHEAD, OP_MW};
  if (m.arch == PROTEA_MODEL_RESNET18) {
    std::vector<int> v;
    for (int l = 0; l < kG_Layers; ++l)
      for (int base : {GI_F, GI_N, GI_NB, GI_NR, GI_W, GI_R}) v.push_back(base + l);
    for (int l = 1; l < kG_Layers; ++l) v.push_back(GI_D + l);
    v.push_back(GI_HEAD);
    return v;
  }
  std::vector<int> v;
  for (int i = 0; i < 7; ++i) v.push_back(RI_F0 + i);
  v.push_back(RI_HEAD);
  for (int i = 0; i < 6; ++i) v.push_back(RI_D1 + i);
  for (int i = 0; i < 7; ++i) v.push_back(RI_W0 + i);
  for (int i = 0; i < 7; ++i) v.push_back(RI_R0 + i);
  return v;
}

// Algorithmic work of one op for one client-step of `r` rows: FLOPs = 2 x useful
// MACs; bytes = compulsory HBM traffic (every operand read once, every result
// written once; weights fp32, activations e bytes).  DESIGN.md "Roofline".
void op_work(const ModelDims& m, int op, uint64_t r, uint64_t e, uint64_t* fl, uint64_t* by);
int op_class(int op) {
  if (op >= GI_F) {
    if (op < GI_N) return PROTEA_OPC_G_FWD;
    if (op < GI_HEAD || (op >= GI_NB && op < GI_D)) return PROTEA_OPC_G_NORM;
    if (op == GI_HEAD) return PROTEA_OPC_G_HEAD;
    if (op < GI_W) return PROTEA_OPC_G_DGRAD;
    if (op < GI_R) return PROTEA_OPC_G_WGRAD;
    return PROTEA_OPC_G_REDUCE;
  }
  if (op < RI_F0) return op;
  if (op < RI_HEAD) return PROTEA_OPC_R_FWD;
  if (op == RI_HEAD) return PROTEA_OPC_R_HEAD;
  if (op < RI_W0) return PROTEA_OPC_R_DGRAD;
  if (op < RI_R0) return PROTEA_OPC_R_WGRAD;
  return PROTEA_OPC_R_REDUCE;
}
void op_work(const ModelDims& m, int op, uint64_t r, uint64_t e, uint64_t* fl, uint64_t* by) {
  if (op >= GI_F) {  // ResNet-18: conv FLOPs = 2 x useful MACs; bytes = operands once + results once
    uint64_t F = 0, B = 0;
    auto conv_io = [&](const Layer& l) {
      return r * (uint64_t)l.hin * l.win * l.cin * e + r * (uint64_t)l.hout * l.wout * l.cout * e;
    };
    if (op == GI_HEAD) {
      F = 3 * 2 * r * 512 * m.classes;
      B = r * 16 * 512 * e * 2 + 8 * m.classes * 513;
    } else if (op < GI_N) {
      const Layer& l = gconv(m, op - GI_F);
      F = 2 * r * l.hout * l.wout * l.cout * 9 * l.cin;
      B = conv_io(l) + 4 * (uint64_t)l.cout * (9 * l.cin + 1);
    } else if (op < GI_HEAD || (op >= GI_NB && op < GI_NR)) {
      const Layer& l = gconv(m, (op < GI_HEAD ? op - GI_N : op - GI_NB));
      B = r * (uint64_t)l.hout * l.wout * l.cout * e * (op < GI_HEAD ? 3 : 5);
    } else if (op < GI_D) {
      const Layer& l = gconv(m, op - GI_NR);
      B = r * 2 * 4 * (uint64_t)l.cout + 16 * (uint64_t)l.cout;
    } else if (op < GI_W) {
      const Layer& l = gconv(m, op - GI_D);
      F = 2 * r * l.hout * l.wout * l.cout * 9 * l.cin;
      B = conv_io(l) + 4 * (uint64_t)l.cout * 9 * l.cin;
    } else if (op < GI_R) {
      const Layer& l = gconv(m, op - GI_W);
      F = 2 * r * l.hout * l.wout * l.cout * 9 * l.cin;
      B = conv_io(l) + 4 * (uint64_t)rsplits(l, (int)r) * l.cout * (9 * l.cin + 1);
    } else {
      const Layer& l = gconv(m, op - GI_R);
      B = 4 * (uint64_t)rsplits(l, (int)r) * l.cout * (9 * l.cin + 1) + 8 * (uint64_t)l.cout * (9 * l.cin + 1);
    }
    *fl = F;
    *by = B;
    return;
  }
  if (op >= RI_F0) {
    uint64_t F = 0, B = 0;
    if (op == RI_HEAD) {
      F = 3 * 2 * r * 64 * m.classes;
      B = r * 4096 * e * 2 + 8 * m.classes * 65 + r * 4;
    } else if (op < RI_HEAD || op < RI_W0) {
      const bool fwd = op < RI_HEAD;
      const Layer& l = m.layers[fwd ? op - RI_F0 : 1 + op - RI_D1];
      F = 2 * r * l.hout * l.wout * l.cout * 9 * l.cin;
      B = r * (uint64_t)l.hin * l.win * l.cin * e + 4 * (uint64_t)l.cout * 9 * l.cin +
          r * (uint64_t)l.hout * l.wout * l.cout * e * 2;
    } else if (op < RI_R0) {
      const Layer& l = m.layers[op - RI_W0];
      F = 2 * r * l.hout * l.wout * l.cout * 9 * l.cin;
      B = r * (uint64_t)l.hin * l.win * l.cin * e + r * (uint64_t)l.hout * l.wout * l.cout * e +
          4 * (uint64_t)r8_split_cap(op - RI_W0, (int)r) * l.cout * (9 * l.cin + 1);
    } else {
      const Layer& l = m.layers[op - RI_R0];
      B = 4 * (uint64_t)r8_split_cap(op - RI_R0, (int)r) * l.cout * (9 * l.cin + 1) +
          8 * (uint64_t)l.cout * (9 * l.cin + 1);
    }
    *fl = F;
    *by = B;
    return;
  }
  const uint64_t c1 = m.c1, c2 = m.c2, f = m.f, C = m.classes;
  // image geometry (CIFAR 32x32x3: HW 1024, HW2 256, HW4 64; FEMNIST 28x28x1: 784, 196, 49)
  const uint64_t HW = (uint64_t)m.H * m.W, HW2 = HW / 4, HW4 = HW / 16, D = HW * m.C, KC = 25 * (uint64_t)m.C;
  const bool tcq = m.width_q == 4 && e == 2 && m.H == 32;
  const uint64_t s1 = tcq ? cdiv((int)r, w1q_ips((int)r)) : cdiv((int)(r * HW), kWgradChunkPx), s2 = cdiv((int)(r * HW2), kWgradChunkPx);
  uint64_t F = 0, B = 0;
  switch (op) {
    case OP_C1F: F = 2 * r * HW * c1 * KC; B = r * D + 4 * c1 * (KC + 1) + r * HW2 * c1 * (e + 1); break;
    case OP_C2F: F = 2 * r * HW2 * c2 * 25 * c1; B = r * HW2 * c1 * e + e * c2 * 25 * c1 + 4 * c2 + r * HW4 * c2 * (e + 1); break;
    case OP_F1F: F = 2 * r * f * HW4 * c2; B = r * HW4 * c2 * e + e * f * HW4 * c2 + 4 * f + r * f * e; break;
    case OP_HEAD: F = 3 * 2 * r * C * f; B = r * f * e + 8 * C * (f + 1) + r * f * e + 8 * f + r * 4; break;
    case OP_F1D: F = 2 * r * HW4 * c2 * f; B = r * f * e + e * f * HW4 * c2 + r * HW4 * c2 * (e + 1) + r * HW2 * c2 * e; break;
    // fp32 master read + write (8 B per weight per client-step) + the dh / a2 reads; the bf16
    // shadow write of the bf16 mode (2 B per weight) is implementation traffic, not counted here
    case OP_F1W: F = 2 * r * f * HW4 * c2; B = r * f * e + r * HW4 * c2 * e + 8 * f * HW4 * c2; break;
    case OP_C2D: F = 2 * r * HW2 * c1 * 25 * c2; B = r * HW2 * c2 * e + e * c2 * 25 * c1 + r * HW2 * c1 * (e + 1) + r * HW * c1 * e; break;
    case OP_C2W: F = 2 * r * HW2 * c2 * 25 * c1; B = r * HW2 * c2 * e + r * HW2 * c1 * e + 4 * s2 * c2 * (25 * c1 + 1); break;
    case OP_C2R: F = 0; B = 4 * s2 * c2 * (25 * c1 + 1) + (8 + (e == 2 ? 2 : 0)) * c2 * (25 * c1 + 1); break;
    case OP_C1W: F = 2 * r * HW * c1 * KC; B = r * HW * c1 * e + r * D + 4 * s1 * c1 * (KC + 1); break;
    case OP_C1R: F = 0; B = 4 * s1 * c1 * (KC + 1) + 8 * c1 * (KC + 1); break;
    case OP_MF: F = 2 * r * 64 * 784; B = r * 784 + 4 * 64 * 785 + r * 64 * e; break;
    case OP_MHEAD: F = 3 * 2 * r * C * 64; B = r * 64 * e + 8 * C * 65 + r * 64 * e + 8 * 64 + r * 4; break;
    case OP_MW: F = 2 * r * 64 * 784; B = r * 64 * e + r * 784 + 8 * 64 * 784; break;
    case OP_STAGE: F = 0; B = r * 3072 + r * 1296 * 16; break;
  }
  *fl = F;
  *by = B;
}

CnnDims cnn_dims(const ModelDims& m) {
  CnnDims d;
  d.c1 = m.c1;
  d.c2 = m.c2;
  d.f = m.f;
  d.classes = m.classes;
  d.w1 = m.layers[0].off_w;
  d.b1 = m.layers[0].off_b;
  d.w2 = m.layers[1].off_w;
  d.b2 = m.layers[1].off_b;
  d.w3 = m.layers[2].off_w;
  d.b3 = m.layers[2].off_b;
  d.w4 = m.layers[3].off_w;
  d.b4 = m.layers[3].off_b;
  d.H = m.H;
  d.W = m.W;
  d.C = m.C;
  return d;
}

MlpDims mlp_dims(const ModelDims& m) {
  MlpDims d;
  d.classes = m.classes;
  d.w1 = m.layers[0].off_w;
  d.b1 = m.layers[0].off_b;
  d.w2 = m.layers[1].off_w;
  d.b2 = m.layers[1].off_b;
  return d;
}

// One (iteration, group) launch descriptor, offsets into the int32 table.
struct Launch {
  int group;
  int vg;  // virtual group = group * lanes + lane: the stream it runs on
  int ntask;
  int64_t task_off;            // tasks: 4 ints each
  int64_t prefix_off[OP_COUNT];
  int grid[OP_COUNT];
  int c2w_groups;                       // width-1 conv2 wgrad: M-tile groups per split (1 or 7)
  int max_rows;                         // largest batch of the launch (grids indexed by client: k_stage_x)
  uint64_t fl[OP_COUNT], by[OP_COUNT];  // algorithmic work of each op of this launch (op_work)
};

template <class OpT, int BM, int BN>
void launch_gemm(protea_ctx* ctx, const OpT& op, const Launch& L, int opid, const int32_t* dtab) {
  const Task* tasks = reinterpret_cast<const Task*>(dtab + L.task_off);
  const int* prefix = dtab + L.prefix_off[opid];
  const int ev = op_begin(ctx, op_class(opid), opid);
  k_gemm_simt<BM, BN, OpT><<<L.grid[opid], (BM / 4) * (BN / 4), 0, ctx->cur>>>(op, tasks, prefix, L.ntask);
  op_end(ctx, ev);
}

template <int BN, int STAGES, class OpT>
void launch_gemm_tc(protea_ctx* ctx, const OpT& op, const Launch& L, int opid, const int32_t* dtab,
                    int smem_floor = 0) {  // smem_floor: reserve at least this much (fewer resident CTAs)
  constexpr int SMEM = tc_smem_bytes<BN, STAGES>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm_tc<BN, STAGES, OpT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  const Task* tasks = reinterpret_cast<const Task*>(dtab + L.task_off);
  const int* prefix = dtab + L.prefix_off[opid];
  const int ev = op_begin(ctx, op_class(opid), opid);
  launch_k(ctx, k_gemm_tc<BN, STAGES, OpT>, L.grid[opid], kTcThreads, (size_t)std::max(SMEM, smem_floor), op, tasks,
           prefix, L.ntask);
  op_end(ctx, ev);
}

int g_num_sms = 148;

template <int BN, int STAGES, class OpT>
void launch_gemm_persistent(protea_ctx* ctx, const OpT& op, const Launch& L, int opid, const int32_t* dtab,
                            int ctas_per_sm) {
  constexpr int SMEM = pers_smem_bytes<BN, STAGES>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm_persistent<BN, STAGES, OpT>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr = true;
  }
  const Task* tasks = reinterpret_cast<const Task*>(dtab + L.task_off);
  const int grid = std::min(L.grid[opid], ctas_per_sm * ctx->spin_cap);
  const int ev = op_begin(ctx, op_class(opid), opid);
  launch_k(ctx, k_gemm_persistent<BN, STAGES, OpT>, grid, kPersThreads, SMEM, op, tasks,
           (const int*)(dtab + L.prefix_off[opid]), L.ntask);
  op_end(ctx, ev);
}

template <class Op>
void launch_conv_persistent(protea_ctx* ctx, const ClientRec* drecs, const CnnDims& d, const Launch& L, int opid,
                            const int32_t* dtab) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_conv_persistent<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, Op::SMEM);
    attr = true;
  }
  Op op;
  op.recs = drecs;
  op.d = d;
  const Task* tasks = reinterpret_cast<const Task*>(dtab + L.task_off);
  // MIN_BLOCKS CTAs per SM (default 1), each a contiguous tile range
  const int per_sm = std::max(1, std::min<int>(min_blocks<Op>::value, (227 * 1024) / (Op::SMEM + 1024)));
  const int grid = std::min(L.grid[opid], per_sm * ctx->spin_cap);
  const int ev = op_begin(ctx, op_class(opid), opid);
  launch_k(ctx, k_conv_persistent<Op>, grid, kConvThreads, Op::SMEM, op, tasks, (const int*)(dtab + L.prefix_off[opid]),
           L.ntask);
  op_end(ctx, ev);
}

void launch_conv1_wgrad_q(protea_ctx* ctx, const ClientRec* drecs, const Launch& L, const int32_t* dtab,
                          const CnnDims& d, float lr) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_conv1_wgrad_q, cudaFuncAttributeMaxDynamicSharedMemorySize, kW1Smem);
    attr = true;
  }
  const Task* tasks = reinterpret_cast<const Task*>(dtab + L.task_off);
  const int grid = std::min(L.grid[OP_C1W], ctx->spin_cap);  // spin-waiting split reduce: all CTAs co-resident
  const int ev = op_begin(ctx, OP_C1W, OP_C1W);
  launch_k(ctx, k_conv1_wgrad_q, grid, kConvThreads, kW1Smem, drecs, tasks, (const int*)(dtab + L.prefix_off[OP_C1W]),
           L.ntask, d.w1, d.b1, lr);
  op_end(ctx, ev);
}

void launch_conv2_wgrad_halo(protea_ctx* ctx, const ClientRec* drecs, const CnnDims& d, const Launch& L,
                             const int32_t* dtab, float lr) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_conv2_wgrad_halo, cudaFuncAttributeMaxDynamicSharedMemorySize, kW2Smem);
    attr = true;
  }
  const Task* tasks = reinterpret_cast<const Task*>(dtab + L.task_off);
  const int grid = std::min(L.grid[OP_C2W], ctx->spin_cap);  // spin-waiting split reduce: all CTAs co-resident
  // deferred split reduce: the weights are next read by the group's next conv2 fwd, so the reduce runs on
  // the low-priority side stream and overlaps conv1 wgrad (single-stream rounds only)
  const int defer = ctx->defer_c2r && ctx->single_chain && ctx->cur == ctx->hi && !ctx->serialize;
  const int ev = op_begin(ctx, OP_C2W, OP_C2W);
  launch_k(ctx, k_conv2_wgrad_halo, grid, kConvThreads, kW2Smem, drecs, tasks, (const int*)(dtab + L.prefix_off[OP_C2W]),
           L.ntask, d, lr, L.c2w_groups, defer);
  op_end(ctx, ev);
  if (defer) {
    cudaEventRecord(ctx->fork_ev, ctx->cur);
    cudaStreamWaitEvent(ctx->side, ctx->fork_ev, 0);
    k_conv2_wgrad_reduce<<<dim3(cdiv(64 * (kW2NP / 4), 256), L.ntask), 256, 0, ctx->side>>>(drecs, tasks, d, lr);
    ctx->launches++;
    cudaEventRecord(ctx->gjoin[L.group], ctx->side);
    ctx->gpending[L.group] = 1;
  }
}

// Evaluate round: the classifier head after the forward kernels (kernels_misc.cuh k_eval_head)
template <typename T>
void launch_eval(protea_ctx* ctx, const Launch& L, const ClientRec* drecs, const Task* tasks, int feat_buf, int F,
                 int hw, const Layer& fc, int C) {
  const int ev = op_begin(ctx, PROTEA_OPC_EVAL_HEAD);
  k_eval_head<T><<<L.ntask, kEvalThreads, 0, ctx->cur>>>(drecs, tasks, feat_buf, F, hw, fc.off_w, fc.off_b, C);
  op_end(ctx, ev);
}

template <typename T>
void launch_head_cnn(protea_ctx* ctx, const ModelDims& m, const Launch& L, const ClientRec* drecs, const Task* tasks,
                     float lr) {
  const CnnDims d = cnn_dims(m);
  const size_t staged = head_cnn_smem_staged(m.f, m.classes, sizeof(T));
  const int stage_h = staged <= kHeadStageMax;
  const size_t smem = stage_h ? staged : head_cnn_smem(m.f, m.classes);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_head_cnn<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kHeadStageMax);
    attr = true;
  }
  HeadArgs ha{drecs, B_H, B_DH, m.f, m.classes, d.w4, d.b4, d.b3, lr};
  const int ev = op_begin(ctx, OP_HEAD, OP_HEAD);
  launch_k(ctx, k_head_cnn<T>, L.ntask, kHeadCnnThreads, smem, ha, tasks, stage_h);
  op_end(ctx, ev);
}

template <class OpT>
OpT tma_op(const ClientRec* recs, const CnnDims& d) {
  OpT op;
  op.recs = recs;
  op.d = d;
  return op;
}
template <class OpT>
OpT tma_op_lr(const ClientRec* recs, const CnnDims& d, float lr) {
  OpT op = tma_op<OpT>(recs, d);
  op.lr = lr;
  return op;
}

// fc1 wgrad op: operands by TMA (TmaFc1Wgrad)
template <int WQ>
TmaFc1Wgrad<WQ> f1w_op(const ClientRec* recs, const CnnDims& d, float lr) {
  TmaFc1Wgrad<WQ> op;
  op.recs = recs;
  op.d = d;
  op.lr = lr;
  return op;
}

// bf16 mode, CNN: conv1, conv2 and fc1 (fwd / dgrad / wgrad) on tcgen05; the head on SIMT
template <int WQ>
void launch_step_tc_w(protea_ctx* ctx, const ModelDims& m, const Launch& L, const ClientRec* drecs,
                      const int32_t* dtab, float lr) {
  typedef __nv_bfloat16 T;
  const Task* tasks = reinterpret_cast<const Task*>(dtab + L.task_off);
  const CnnDims d = cnn_dims(m);
  int ev = op_begin(ctx, OP_STAGE, OP_STAGE);
  launch_k(ctx, k_stage_x, dim3(cdiv(L.max_rows * 1296, kStageThreads * kStagePx), L.ntask), kStageThreads, 0, drecs, tasks);
  op_end(ctx, ev);
  launch_conv_persistent<QuadConv1<WQ>>(ctx, drecs, d, L, OP_C1F, dtab);
  join_group(ctx, L.group);  // the previous step's deferred fc1 wgrad still reads a2
  if constexpr (WQ == 4)
    launch_conv_persistent<HaloConv2Q<false>>(ctx, drecs, d, L, OP_C2F, dtab);
  else if constexpr (WQ == 2)
    launch_conv_persistent<HaloConv2<WQ, false>>(ctx, drecs, d, L, OP_C2F, dtab);
  else
    launch_gemm_tc<TC_C2F_BN, TC_STAGES>(ctx, TmaConv2Fwd<WQ>{drecs, d}, L, OP_C2F, dtab);
  // (a split-K persistent variant for light iterations measured slower: 7.2 -> 8.0 ms/round)
  launch_gemm_tc<TC_F1F_BN, TC_F1F_STAGES>(ctx, tma_op<TmaFc1Fwd<WQ>>(drecs, d), L, OP_F1F, dtab);
  if (ctx->eval_mode) {
    launch_eval<T>(ctx, L, drecs, tasks, B_H, m.f, 1, m.layers[3], m.classes);
    return;
  }
  launch_head_cnn<T>(ctx, m, L, drecs, tasks, lr);
  launch_gemm_persistent<TC_F1D_BN, 8>(ctx, tma_op<TmaFc1Dgrad<WQ>>(drecs, d), L, OP_F1D, dtab, 1);
  // fc1 wgrad (HBM-bound RMW of the fp32 master + bf16 shadow) needs dh, a2 and the fc1 weights, which
  // nothing in the rest of this step touches.  In light iterations (the lock-step tail, where every
  // other op is latency bound) it runs on the low-priority side stream and is joined only before the
  // next conv2 fwd of the group (which overwrites a2), a release, or the end of the round.
  if (ctx->overlap_now) {
    cudaEventRecord(ctx->fork_ev, ctx->cur);
    cudaStreamWaitEvent(ctx->side, ctx->fork_ev, 0);
    cudaStream_t main = ctx->cur;
    ctx->cur = ctx->side;
    // deferred: fewer resident CTAs (PROTEA_F1W_SIDE_SMEM) spread its HBM stream over the chain it overlaps
    launch_gemm_tc<TC_F1W_BN, TC_F1W_STAGES>(ctx, f1w_op<WQ>(drecs, d, lr), L, OP_F1W, dtab, ctx->f1w_side_smem);
    cudaEventRecord(ctx->gjoin[L.group], ctx->side);
    ctx->gpending[L.group] = 1;
    ctx->cur = main;
  } else {
    launch_gemm_tc<TC_F1W_BN, TC_F1W_STAGES>(ctx, f1w_op<WQ>(drecs, d, lr), L, OP_F1W, dtab);
  }
  if constexpr (WQ == 4)
    launch_conv_persistent<HaloConv2Q<true>>(ctx, drecs, d, L, OP_C2D, dtab);
  else
    launch_conv_persistent<HaloConv2<WQ, true>>(ctx, drecs, d, L, OP_C2D, dtab);
  if constexpr (WQ == 4)
    launch_conv2_wgrad_halo(ctx, drecs, d, L, dtab, lr);
  else
    launch_gemm_tc<TC_C2W_BN, TC_STAGES>(ctx, tma_op_lr<TmaConv2Wgrad<WQ>>(drecs, d, lr), L, OP_C2W, dtab);

  if constexpr (WQ == 4) {
    launch_conv1_wgrad_q(ctx, drecs, L, dtab, d, lr);  // the split reduce + SGD is fused (last split)
  } else {
    launch_gemm_tc<TC_C1W_BN, TC_STAGES>(ctx, TcConv1Wgrad<WQ>{drecs, d}, L, OP_C1W, dtab);
    ev = op_begin(ctx, OP_C1R, OP_C1R);
    k_reduce_conv1_tc<<<L.grid[OP_C1R], kReduceBlock, 0, ctx->cur>>>(drecs, tasks, dtab + L.prefix_off[OP_C1R],
                                                                         L.ntask, m.c1, d.w1, d.b1, lr);
    op_end(ctx, ev);
  }
}

void launch_step_tc(protea_ctx* ctx, const ModelDims& m, const Launch& L, const ClientRec* drecs, const int32_t* dtab,
                    float lr) {
  if (m.width_q == 1)
    launch_step_tc_w<1>(ctx, m, L, drecs, dtab, lr);
  else if (m.width_q == 2)
    launch_step_tc_w<2>(ctx, m, L, drecs, dtab, lr);
  else
    launch_step_tc_w<4>(ctx, m, L, drecs, dtab, lr);
}

int ilog2(int v) {
  int r = 0;
  while ((1 << (r + 1)) <= v) ++r;
  return r;
}
RTcConv rtc(const Layer& l) {
  RTcConv c;
  c.H = l.hin;
  c.W = l.win;
  c.Cin = l.cin;
  c.Cout = l.cout;
  c.s = l.stride;
  c.Ho = l.hout;
  c.Wo = l.wout;
  c.lci = ilog2(l.cin);
  c.lco = ilog2(l.cout);
  c.lw = ilog2(l.win);
  c.lhw = ilog2(l.hin * l.win);
  c.lwo = ilog2(l.wout);
  c.lhwo = ilog2(l.hout * l.wout);
  c.w = l.off_w;
  c.b = l.off_b;
  return c;
}

RConv rconv(const Layer& l) {
  RConv c;
  c.H = l.hin;
  c.W = l.win;
  c.Cin = l.cin;
  c.Cout = l.cout;
  c.s = l.stride;
  c.Ho = l.hout;
  c.Wo = l.wout;
  c.w = l.off_w;
  c.b = l.off_b;
  return c;
}

// ResNet tcgen05 ops: persistent cp.async GEMM, contiguous tile ranges; the B tile (BN) sized to the
// layer's N (16 / 32 -> 32, 64 -> 64) so no gather slots are spent on zero-filled columns
template <int BN, class Op>
void launch_rtc_bn(protea_ctx* ctx, const Op& op, const Launch& L, int opid, const int32_t* dtab, int sm_cap) {
  constexpr int RS = 8;  // ring stages (1 CTA per SM: 8 K blocks in flight)
  constexpr int SMEM = rp_smem_bytes<BN, RS>();
  static int per_sm = 0;  // resident CTAs per SM (registers / shared memory): the persistent grid
  if (!per_sm) {
    cudaFuncSetAttribute(k_gemm_tc_pers<BN, RS, Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gemm_tc_pers<BN, RS, Op>, kRpThreads, SMEM);
    per_sm = std::max(1, std::min(per_sm, 2));
  }
  const Task* tasks = reinterpret_cast<const Task*>(dtab + L.task_off);
  const int grid = std::min(L.grid[opid], per_sm * sm_cap);
  const int ev = op_begin(ctx, op_class(opid), opid);
  launch_k(ctx, k_gemm_tc_pers<BN, RS, Op>, grid, kRpThreads, SMEM, op, tasks, (const int*)(dtab + L.prefix_off[opid]),
           L.ntask);
  op_end(ctx, ev);
}
template <class Op>
void launch_rtc(protea_ctx* ctx, const Op& op, const Launch& L, int opid, const int32_t* dtab, int N,
                int sm_cap = 0) {
  if (sm_cap <= 0) sm_cap = g_num_sms;
  if (N <= 32)
    launch_rtc_bn<32>(ctx, op, L, opid, dtab, sm_cap);
  else
    launch_rtc_bn<64>(ctx, op, L, opid, dtab, sm_cap);
}

// Persistent conv op (k_conv_persistent) over min(tiles, resident CTAs per SM x SMs) CTAs; sm_cap as
// launch_rtc (an SM share for concurrent streams)
template <class Op>
void launch_conv_op(protea_ctx* ctx, const Op& op, const Launch& L, int opid, const int32_t* dtab, int sm_cap) {
  static int per_sm = 0;
  if (!per_sm) {
    cudaFuncSetAttribute(k_conv_persistent<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, Op::SMEM);
    // without a carveout preference the occupancy query (and the launch) may assume a smaller shared-memory
    // partition: 1 resident CTA where the op is built for MIN_BLOCKS
    cudaFuncSetAttribute(k_conv_persistent<Op>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    const cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_conv_persistent<Op>, kConvThreads, Op::SMEM);
    if (std::getenv("PROTEA_VERBOSE")) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, k_conv_persistent<Op>);
      fprintf(stderr, "launch_conv_op %s: occupancy rc %d per_sm %d smem %d regs %d static_smem %zu local %zu maxthr %d maxdyn %d carve %d\n",
              __PRETTY_FUNCTION__, (int)oe, per_sm, Op::SMEM, fa.numRegs, fa.sharedSizeBytes, fa.localSizeBytes,
              fa.maxThreadsPerBlock, fa.maxDynamicSharedSizeBytes, fa.preferredShmemCarveout);
    }
    // the occupancy query reports 1 CTA per SM for these tcgen05 kernels even where registers (launch bounds
    // MIN_BLOCKS) and shared memory admit more (measured: RHalo<16> 64 regs x 320 threads, 43 KB): size the
    // grid from the kernel's own limits (TMEM is allocated per CTA and fits MIN_BLOCKS x TMEM_COLS <= 512)
    per_sm = std::max(per_sm, std::min<int>(min_blocks<Op>::value, (227 * 1024) / (Op::SMEM + 1024)));
    if (const char* cap = std::getenv("PROTEA_CONV_PER_SM")) per_sm = std::min(per_sm, std::atoi(cap));
    if (oe != cudaSuccess || per_sm < 1) per_sm = 1;
  }
  const Task* tasks = reinterpret_cast<const Task*>(dtab + L.task_off);
  const int grid = std::min(L.grid[opid], per_sm * std::min(sm_cap > 0 ? sm_cap : g_num_sms, ctx->spin_cap));
  const int ev = op_begin(ctx, op_class(opid), opid);
  launch_k(ctx, k_conv_persistent<Op>, grid, kConvThreads, Op::SMEM, op, tasks,
           (const int*)(dtab + L.prefix_off[opid]), L.ntask);
  op_end(ctx, ev);
}
// ResNet-8 stride-1 layer on the halo kernel (kernels_resnet_halo.cuh)
template <int C, bool DGRAD>
void launch_r8_halo_c(protea_ctx* ctx, RHalo<C, DGRAD> op, const Launch& L, int opid, const int32_t* dtab,
                      int sm_cap) {
  launch_conv_op(ctx, op, L, opid, dtab, sm_cap);
}
template <class P>
void launch_r8_wgrad_halo_p(protea_ctx* ctx, const ClientRec* drecs, int i, int in_tm, int dout_tm, const Launch& L,
                            int opid, const int32_t* dtab, int sm_cap) {
  static int per_sm = 0;
  if (!per_sm) {
    cudaFuncSetAttribute(k_r8_wgrad_halo<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, P::SMEM);
    cudaFuncSetAttribute(k_r8_wgrad_halo<P>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    const cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_r8_wgrad_halo<P>, kConvThreads, P::SMEM);
    if (std::getenv("PROTEA_VERBOSE"))
      fprintf(stderr, "launch_r8_wgrad_halo %s: occupancy rc %d per_sm %d smem %d\n", __PRETTY_FUNCTION__, (int)oe, per_sm, P::SMEM);
    per_sm = std::max(per_sm, std::min<int>(P::TMEM_COLS <= 256 ? 2 : 1, (227 * 1024) / (P::SMEM + 1024)));  // (as launch_conv_op)
    if (const char* cap = std::getenv("PROTEA_WG_PER_SM")) per_sm = std::min(per_sm, std::atoi(cap));
    if (oe != cudaSuccess || per_sm < 1) per_sm = 1;
    per_sm = std::min(per_sm, 512 / P::TMEM_COLS);  // resident CTAs must fit their TMEM allocations
  }
  const Task* tasks = reinterpret_cast<const Task*>(dtab + L.task_off);
  const int grid = std::min(L.grid[opid], per_sm * (sm_cap > 0 ? sm_cap : g_num_sms));
  const int ev = op_begin(ctx, op_class(opid), opid);
  launch_k(ctx, k_r8_wgrad_halo<P>, grid, kConvThreads, P::SMEM, drecs, tasks, (const int*)(dtab + L.prefix_off[opid]),
           L.ntask, in_tm, dout_tm, i);
  op_end(ctx, ev);
}
// layer index i in {1, 2, 4, 6}: map slot k = 0..3
int r8_halo_slot(int i) { return i == 1 ? 0 : i == 2 ? 1 : i == 4 ? 2 : 3; }
void launch_r8_wgrad_halo(protea_ctx* ctx, const ClientRec* drecs, const Layer& l, int i, const Launch& L, int opid,
                          const int32_t* dtab, int sm_cap = 0) {
  if (i == 0) {
    launch_r8_wgrad_halo_p<RWgHalo0>(ctx, drecs, 0, RTM_IN0, RTM_WD0, L, opid, dtab, sm_cap);
    return;
  }
  if (l.stride == 2) {
    const int k = i == 3 ? 0 : 1;
    if (l.cin == 16) launch_r8_wgrad_halo_p<RWgHaloS2<16>>(ctx, drecs, i, RTM_IN3 + k, RTM_WD3 + k, L, opid, dtab, sm_cap);
    else launch_r8_wgrad_halo_p<RWgHaloS2<32>>(ctx, drecs, i, RTM_IN3 + k, RTM_WD3 + k, L, opid, dtab, sm_cap);
    return;
  }
  const int k = r8_halo_slot(i);
  if (l.cin == 16) launch_r8_wgrad_halo_p<RWgHalo<16>>(ctx, drecs, i, RTM_IN1 + k, RTM_WD1 + k, L, opid, dtab, sm_cap);
  else if (l.cin == 32) launch_r8_wgrad_halo_p<RWgHalo<32>>(ctx, drecs, i, RTM_IN1 + k, RTM_WD1 + k, L, opid, dtab, sm_cap);
  else launch_r8_wgrad_halo_p<RWgHalo<64>>(ctx, drecs, i, RTM_IN1 + k, RTM_WD1 + k, L, opid, dtab, sm_cap);
}
void launch_r8_halo_s2(protea_ctx* ctx, const ClientRec* drecs, const Layer& l, int i, int out_buf, const Launch& L,
                       int opid, const int32_t* dtab) {
  const int k = i == 3 ? 0 : 1;
  if (l.cin == 16)
    launch_conv_op(ctx, RHaloS2<16>{drecs, RTM_IN3 + k, RTM_W3 + k, out_buf, l.off_b}, L, opid, dtab, 0);
  else
    launch_conv_op(ctx, RHaloS2<32>{drecs, RTM_IN3 + k, RTM_W3 + k, out_buf, l.off_b}, L, opid, dtab, 0);
}
template <bool DGRAD>
void launch_r8_halo(protea_ctx* ctx, const ClientRec* drecs, const Layer& l, int i, int out_buf, int res_buf,
                    int res_mode, int Cres, int mask_buf, const Launch& L, int opid, const int32_t* dtab,
                    int sm_cap = 0) {
  const int k = r8_halo_slot(i);
  const int in_tm = (DGRAD ? RTM_DO1 : RTM_IN1) + k, w_tm = RTM_W1 + k;
  switch (l.cin) {
    case 16: launch_r8_halo_c<16, DGRAD>(ctx, {drecs, in_tm, w_tm, out_buf, res_buf, res_mode, Cres, mask_buf, l.off_b},
                                         L, opid, dtab, sm_cap); break;
    case 32: launch_r8_halo_c<32, DGRAD>(ctx, {drecs, in_tm, w_tm, out_buf, res_buf, res_mode, Cres, mask_buf, l.off_b},
                                         L, opid, dtab, sm_cap); break;
    default: launch_r8_halo_c<64, DGRAD>(ctx, {drecs, in_tm, w_tm, out_buf, res_buf, res_mode, Cres, mask_buf, l.off_b},
                                         L, opid, dtab, sm_cap); break;
  }
}

void stage_r(protea_ctx* ctx, const ClientRec* drecs, const Task* tasks, const Launch& L, int out_buf) {
  const int ev = op_begin(ctx, PROTEA_OPC_R_FWD);
  k_stage_r<<<dim3(L.ntask, 16), 256, 0, ctx->cur>>>(drecs, tasks, out_buf);
  op_end(ctx, ev);
}

// ResNet-8 step (fp32 verify: SIMT; bf16 mode: tcgen05 convs, kernels_resnet_tc.cuh, activations in bf16).  Buffers: a0 r1 o1 r2 o2 r3 o3, gradients
// ping-pong g0 g1 g2; each layer's dgrad runs before its SGD update (old weights).
template <typename T>
void launch_step_resnet(protea_ctx* ctx, const ModelDims& m, const Launch& L, const ClientRec* drecs,
                        const int32_t* dtab, float lr) {
  const Task* tasks = reinterpret_cast<const Task*>(dtab + L.task_off);
  const int in_of[7] = {-1, B_R_A0, B_R_R1, B_R_O1, B_R_R2, B_R_O2, B_R_R3};
  const int out_of[7] = {B_R_A0, B_R_R1, B_R_O1, B_R_R2, B_R_O2, B_R_R3, B_R_O3};
  typedef RFwd<T, R_BM, R_BN> F;
  typedef RDgrad<T, R_BM, R_BN> D;
  typedef RWgrad<T, R_BM, R_BN> Wg;
  constexpr bool TC = std::is_same<T, __nv_bfloat16>::value;  // bf16 mode: layers 1-6 on tcgen05
  for (int i = 0; i < 7; ++i) {
    F f;
    f.recs = drecs;
    f.L = rconv(m.layers[i]);
    f.in_buf = in_of[i];
    f.out_buf = out_of[i];
    f.res_buf = -1;
    f.res_mode = 0;
    f.Cres = 0;
    if (i == 2) { f.res_buf = B_R_A0; f.res_mode = 1; }                      // block 1: identity shortcut
    if (i == 4) { f.res_buf = B_R_O1; f.res_mode = 2; f.Cres = 16; }         // block 2: option A from o1
    if (i == 6) { f.res_buf = B_R_O2; f.res_mode = 2; f.Cres = 32; }         // block 3: option A from o2
    if (TC) {
      RTcFwd tf{drecs, rtc(m.layers[i]), f.in_buf, f.out_buf, f.res_buf, f.res_mode, f.Cres, B_WSH};
      if (i == 0) {  // conv0: the u8 input staged once per step as [r][32][32][8] bf16 (xs)
        stage_r(ctx, drecs, tasks, L, B_R_XS);
        tf.L.Cin = 8;
        tf.L.lci = 3;
        tf.in_buf = B_R_XS;
        tf.wbuf = B_R_W0P;
      }
      if (i == 0 && r8_halo0(m.layers[0], R8H_FWD))
        launch_conv_op(ctx, RHalo0{drecs, f.out_buf, m.layers[0].off_b}, L, RI_F0, dtab, 0);
      else if (r8_halo_s2(m.layers[i]))
        launch_r8_halo_s2(ctx, drecs, m.layers[i], i, f.out_buf, L, RI_F0 + i, dtab);
      else if (r8_halo_c(m.layers[i], R8H_FWD))
        launch_r8_halo<false>(ctx, drecs, m.layers[i], i, f.out_buf, f.res_buf, f.res_mode, f.Cres, -1, L, RI_F0 + i,
                              dtab);
      else
        launch_rtc(ctx, tf, L, RI_F0 + i, dtab, tf.L.Cout);
      continue;
    }
    launch_gemm<F, R_BM, R_BN>(ctx, f, L, RI_F0 + i, dtab);
  }
  const Layer& fc = m.layers[7];
  if (ctx->eval_mode) {
    launch_eval<T>(ctx, L, drecs, tasks, B_R_O3, 64, 64, fc, m.classes);
    return;
  }
  RHeadArgs ha{drecs, m.classes, fc.off_w, fc.off_b, lr};
  int ev = op_begin(ctx, PROTEA_OPC_R_HEAD, RI_HEAD);
  static bool rh_attr = false;
  if (!rh_attr) {  // classes <= 64: up to 49.4 KB of dynamic shared memory
    cudaFuncSetAttribute(k_rhead<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rhead_smem(64));
    cudaFuncSetAttribute(k_rhead<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rhead_smem(64));
    rh_attr = true;
  }
  k_rhead<T><<<L.ntask, 256, rhead_smem(m.classes), ctx->cur>>>(ha, tasks);
  op_end(ctx, ev);
  // backward, layer 6 (b3b) down to 1 (b1a): dgrad (dout, out, mask, add), then wgrad + reduce
  struct Bw { int dout, out, mask, add, add_mode, cadd; };
  const Bw bw[7] = {
      {0, 0, 0, 0, 0, 0},                              // conv0: no dgrad
      {B_R_G2, B_R_G0, B_R_A0, B_R_G1, 1, 16},         // b1a: dz0 = (convT(dr1) + ds1) * (a0 > 0)
      {B_R_G1, B_R_G2, B_R_R1, -1, 0, 0},              // b1b: dr1 = convT(ds1) * (r1 > 0)
      {B_R_G0, B_R_G1, B_R_O1, B_R_G2, 2, 32},         // b2a: ds1 = (convT_s2(dr2) + sc(ds2)) * (o1 > 0)
      {B_R_G2, B_R_G0, B_R_R2, -1, 0, 0},              // b2b: dr2 = convT(ds2) * (r2 > 0)
      {B_R_G1, B_R_G2, B_R_O2, B_R_G0, 2, 64},         // b3a: ds2 = (convT_s2(dr3) + sc(ds3)) * (o2 > 0)
      {B_R_G0, B_R_G1, B_R_R3, -1, 0, 0}};             // b3b: dr3 = convT(ds3) * (r3 > 0)
  const int wg_dout[7] = {B_R_G0, B_R_G2, B_R_G1, B_R_G0, B_R_G2, B_R_G1, B_R_G0};
  ReduceMultiV rm;
  rm.chunk_base[0] = 0;
  // bf16, one chain: wgrad(i) runs on ctx->wstream beside dgrad(i) (both only read dout(i)), each on half
  // the SMs; the gradient buffers rotate over three, so dgrad(i - 2) (which overwrites wgrad(i)'s dout)
  // waits for wgrad(i), and the merged reduce waits for all of them
  const bool ovl = TC && ctx->r8_overlap && ctx->single_chain && !ctx->serialize && ctx->cur == ctx->hi &&
                   ctx->rows_now <= ctx->r8_overlap_rows;  // light iterations: latency-bound kernels
  const int half = ovl ? std::max(1, g_num_sms / 2) : 0;
  if (ovl)
    for (auto& e : ctx->r8ev)
      if (!e) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  cudaStream_t main_s = ctx->cur;
  for (int i = 6; i >= 0; --i) {
    const Layer& l = m.layers[i];
    if (ovl) {
      cudaEventRecord(ctx->r8ev[8 + i], main_s);  // dout(i) is ready (written before this point)
      if (i + 2 <= 6) cudaStreamWaitEvent(main_s, ctx->r8ev[i + 2], 0);  // wgrad(i + 2) read what dgrad(i) overwrites
    }
    if (i >= 1) {
      D dg;
      dg.recs = drecs;
      dg.L = rconv(l);
      dg.dout_buf = bw[i].dout;
      dg.out_buf = bw[i].out;
      dg.mask_buf = bw[i].mask;
      dg.add_buf = bw[i].add;
      dg.add_mode = bw[i].add_mode;
      dg.Cadd = bw[i].cadd;
      if (TC) {
        RTcDgrad td{drecs, rtc(l), dg.dout_buf, dg.out_buf, dg.mask_buf, dg.add_buf, dg.add_mode, dg.Cadd};
        if (r8_halo_s2(l, R8H_DGRAD)) {
          const int k = i == 3 ? 0 : 1;
          if (l.cin == 16)
            launch_conv_op(ctx, RHaloS2D<16>{drecs, RTM_DO3 + k, RTM_W3 + k, dg.out_buf, dg.add_buf, dg.Cadd, dg.mask_buf},
                           L, RI_D1 + i - 1, dtab, half);
          else
            launch_conv_op(ctx, RHaloS2D<32>{drecs, RTM_DO3 + k, RTM_W3 + k, dg.out_buf, dg.add_buf, dg.Cadd, dg.mask_buf},
                           L, RI_D1 + i - 1, dtab, half);
        } else if (r8_halo_c(l, R8H_DGRAD))  // (the dout halo maps follow this rotation: build_r8_tmaps)
          launch_r8_halo<true>(ctx, drecs, l, i, dg.out_buf, dg.add_buf, dg.add_mode, dg.Cadd, dg.mask_buf, L,
                               RI_D1 + i - 1, dtab, half);
        else
          launch_rtc(ctx, td, L, RI_D1 + i - 1, dtab, td.L.Cin, half);
      } else {
        launch_gemm<D, R_BM, R_BN>(ctx, dg, L, RI_D1 + i - 1, dtab);
      }
    }
    if (TC) {
      RTcWgrad tw{drecs, rtc(l), wg_dout[i], in_of[i], l.cin, i};
      if (i == 0) {  // conv0: the staged input of the forward
        tw.L.Cin = 8;
        tw.L.lci = 3;
        tw.in_buf = B_R_XS;
      }
      const bool hw = r8_halo_c(l, R8H_WGRAD) != 0 || r8_halo_s2(l, R8H_WGRAD) != 0 || r8_halo0(l, R8H_WGRAD);
      if (ovl) {
        ctx->cur = ctx->wstream;
        cudaStreamWaitEvent(ctx->cur, ctx->r8ev[8 + i], 0);
        if (hw) launch_r8_wgrad_halo(ctx, drecs, l, i, L, RI_W0 + i, dtab, g_num_sms - half);
        else launch_rtc(ctx, tw, L, RI_W0 + i, dtab, tw.L.Cout, g_num_sms - half);
        cudaEventRecord(ctx->r8ev[i], ctx->cur);
        ctx->cur = main_s;
      } else {
        if (hw) launch_r8_wgrad_halo(ctx, drecs, l, i, L, RI_W0 + i, dtab);
        else launch_rtc(ctx, tw, L, RI_W0 + i, dtab, tw.L.Cout);
      }
    } else {
      Wg wg;
      wg.recs = drecs;
      wg.L = rconv(l);
      wg.dout_buf = wg_dout[i];
      wg.in_buf = in_of[i];
      wg.layer = i;
      launch_gemm<Wg, R_BM, R_BN>(ctx, wg, L, RI_W0 + i, dtab);
    }
    // SGD of the fp32 master and (bf16 mode) the tensor-core shadow: deferred to one launch after the
    // backward (each layer's dgrad above has read its old weights; the next writer is the next step)
    rm.a[i] = ReduceArgs{drecs, B_R_WSP, l.cout, 9 * l.cin, l.off_w, l.off_b, l.hout * l.wout, lr,
                         TC ? (i == 0 ? 2 : 1) : 0, i};
  }
  if (ovl)
    for (int i = 0; i < 2; ++i) cudaStreamWaitEvent(main_s, ctx->r8ev[i], 0);  // wgrads 2..6 joined above
  for (int i = 0; i < 7; ++i)
    rm.chunk_base[i + 1] = rm.chunk_base[i] + cdiv(m.layers[i].cout * (9 * m.layers[i].cin + 1), 4 * kReduceBlock);
  ev = op_begin(ctx, PROTEA_OPC_R_REDUCE, -1);
  k_reduce_multi_v4<<<dim3(rm.chunk_base[7], L.ntask), kReduceBlock, 0, ctx->cur>>>(rm, tasks);
  op_end(ctx, ev);
}

// ResNet-18 with GroupNorm (R26), SIMT kernels: forward (conv -> GroupNorm [+ shortcut] -> ReLU per layer),
// head, then per block in reverse: GroupNorm bwd (b) -> conv dgrad (b, pre-update W) -> wgrad + SGD (b) ->
// GroupNorm bwd (a) -> dgrad (a, + the shortcut gradient) -> wgrad + SGD (a); the stem last.  Gradient
// buffers: X = d(block output / current activation), YG = d(conv output), ZG = the shortcut gradient.
template <typename T>
void launch_step_r18(protea_ctx* ctx, const ModelDims& m, const Launch& L, const ClientRec* drecs,
                     const int32_t* dtab, float lr) {
  const Task* tasks = reinterpret_cast<const Task*>(dtab + L.task_off);
  typedef RFwd<T, R_BM, R_BN> F;
  typedef RDgrad<T, R_BM, R_BN> D;
  typedef RWgrad<T, R_BM, R_BN> Wg;
  auto prefix = [&](int op) { return (const int*)(dtab + L.prefix_off[op]); };
  auto gn_args = [&](int l) {
    const Layer& c = gconv(m, l);
    const Layer& g = gnorm_of(m, l);
    GnArgs a{};
    a.recs = drecs;
    a.layer = l;
    a.HW = c.hout * c.wout;
    a.C = c.cout;
    a.Wo = c.wout;
    a.z_buf = B_G_Z0 + l;
    a.y_buf = B_G_Y0 + l;
    a.gam = g.off_w;
    a.bet = g.off_b;
    a.res_mode = 0;
    a.res_buf = -1;
    a.gs_buf = -1;
    return a;
  };
  auto conv_fwd = [&](int l, int in_buf) {
    F f;
    f.recs = drecs;
    f.L = rconv(gconv(m, l));
    f.in_buf = in_buf;
    f.out_buf = B_G_Z0 + l;
    f.res_buf = -1;
    f.res_mode = 0;
    f.Cres = 0;
    f.relu = 0;
    launch_gemm<F, R_BM, R_BN>(ctx, f, L, GI_F + l, dtab);
  };
  auto gn_fwd = [&](const GnArgs& a) {
    const int ev = op_begin(ctx, PROTEA_OPC_G_NORM, GI_N + a.layer);
    k_gn_fwd<T><<<L.grid[GI_N + a.layer], kGnThreads, 0, ctx->cur>>>(a, tasks, prefix(GI_N + a.layer), L.ntask);
    op_end(ctx, ev);
  };
  auto gn_bwd = [&](const GnArgs& a) {
    int ev = op_begin(ctx, PROTEA_OPC_G_NORM, GI_NB + a.layer);
    k_gn_bwd<T><<<L.grid[GI_NB + a.layer], kGnThreads, 0, ctx->cur>>>(a, tasks, prefix(GI_NB + a.layer), L.ntask);
    op_end(ctx, ev);
    const Layer& g = gnorm_of(m, a.layer);
    ev = op_begin(ctx, PROTEA_OPC_G_NORM, GI_NR + a.layer);
    k_gn_reduce<<<L.ntask, 256, 0, ctx->cur>>>(drecs, tasks, g.cout, g.off_w, g.off_b, lr);
    op_end(ctx, ev);
  };
  auto wgrad_sgd = [&](int l, int dout_buf, int in_buf) {
    Wg wg;
    wg.recs = drecs;
    wg.L = rconv(gconv(m, l));
    wg.dout_buf = dout_buf;
    wg.in_buf = in_buf;
    wg.layer = -1;
    wg.wsp_buf = B_G_WSP;
    launch_gemm<Wg, R_BM, R_BN>(ctx, wg, L, GI_W + l, dtab);
    const Layer& c = gconv(m, l);
    ReduceArgs ra{drecs, B_G_WSP, c.cout, 9 * c.cin, c.off_w, c.off_b, c.hout * c.wout, lr, 0, -1};
    const int ev = op_begin(ctx, PROTEA_OPC_G_REDUCE, GI_R + l);
    k_reduce_update<<<L.grid[GI_R + l], kReduceBlock, 0, ctx->cur>>>(ra, tasks, prefix(GI_R + l), L.ntask);
    op_end(ctx, ev);
  };
  auto dgrad = [&](int l, int add_buf, int add_mode, int Cadd) {
    D dg;
    dg.recs = drecs;
    dg.L = rconv(gconv(m, l));
    dg.dout_buf = B_G_YG;
    dg.out_buf = B_G_X;
    dg.mask_buf = -1;
    dg.add_buf = add_buf;
    dg.add_mode = add_mode;
    dg.Cadd = Cadd;
    launch_gemm<D, R_BM, R_BN>(ctx, dg, L, GI_D + l, dtab);
  };
  // ---- forward
  conv_fwd(0, -1);
  gn_fwd(gn_args(0));
  for (int i = 0; i < 8; ++i) {
    const int la = 1 + 2 * i, lb = 2 + 2 * i, in_act = B_G_Y0 + 2 * i;
    conv_fwd(la, in_act);
    gn_fwd(gn_args(la));
    conv_fwd(lb, B_G_Y0 + la);
    GnArgs a = gn_args(lb);
    const Layer& ca = gconv(m, la);
    a.res_buf = in_act;
    a.res_mode = (ca.stride == 1 && ca.cin == ca.cout) ? 1 : 2;
    a.Cres = ca.cin;
    gn_fwd(a);
  }
  const Layer& fc = m.layers.back();
  if (ctx->eval_mode) {
    launch_eval<T>(ctx, L, drecs, tasks, B_G_Y0 + 16, 512, 16, fc, m.classes);
    return;
  }
  {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_g_head<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g_head_smem(64));
      attr = true;
    }
    GHeadArgs ha{drecs, m.classes, fc.off_w, fc.off_b, lr, B_G_Y0 + 16, B_G_X};
    const int ev = op_begin(ctx, PROTEA_OPC_G_HEAD, GI_HEAD);
    k_g_head<T><<<L.ntask, 256, g_head_smem(m.classes), ctx->cur>>>(ha, tasks);
    op_end(ctx, ev);
  }
  // ---- backward (X holds d(block output))
  for (int i = 7; i >= 0; --i) {
    const int la = 1 + 2 * i, lb = 2 + 2 * i, in_act = B_G_Y0 + 2 * i;
    const Layer& ca = gconv(m, la);
    GnArgs b = gn_args(lb);
    b.dout_buf = B_G_X;
    b.dz_buf = B_G_YG;
    b.gs_buf = B_G_ZG;
    gn_bwd(b);
    dgrad(lb, -1, 0, 0);                       // d(ra) -> X (pre-update W of conv b)
    wgrad_sgd(lb, B_G_YG, B_G_Y0 + la);
    GnArgs a = gn_args(la);
    a.dout_buf = B_G_X;
    a.dz_buf = B_G_YG;
    gn_bwd(a);
    const bool ident = ca.stride == 1 && ca.cin == ca.cout;
    dgrad(la, B_G_ZG, ident ? 1 : 2, ca.cout);  // d(block input) = convT(dz_a) + shortcut gradient -> X
    wgrad_sgd(la, B_G_YG, in_act);
  }
  GnArgs a0 = gn_args(0);
  a0.dout_buf = B_G_X;
  a0.dz_buf = B_G_YG;
  gn_bwd(a0);
  wgrad_sgd(0, B_G_YG, -1);
}

template <typename T>
void launch_step(protea_ctx* ctx, const ModelDims& m, const Launch& L, const ClientRec* drecs, const int32_t* dtab,
                 float lr) {
  if (m.arch == PROTEA_MODEL_RESNET18) {
    launch_step_r18<T>(ctx, m, L, drecs, dtab, lr);
    return;
  }
  if (m.arch == PROTEA_MODEL_RESNET8) {
    launch_step_resnet<T>(ctx, m, L, drecs, dtab, lr);
    return;
  }
  const Task* tasks = reinterpret_cast<const Task*>(dtab + L.task_off);
  if (m.arch == PROTEA_MODEL_CNN) {
    const CnnDims d = cnn_dims(m);
    launch_gemm<Conv1Fwd<T, C1F_BM, C1F_BN>, C1F_BM, C1F_BN>(ctx, {drecs, d}, L, OP_C1F, dtab);
    launch_gemm<Conv2Fwd<T, C2F_BM, C2F_BN>, C2F_BM, C2F_BN>(ctx, {drecs, d}, L, OP_C2F, dtab);
    launch_gemm<Fc1Fwd<T, F1F_BM, F1F_BN>, F1F_BM, F1F_BN>(ctx, {drecs, d}, L, OP_F1F, dtab);
    if (ctx->eval_mode) {
      launch_eval<T>(ctx, L, drecs, tasks, B_H, m.f, 1, m.layers[3], m.classes);
      return;
    }
    launch_head_cnn<T>(ctx, m, L, drecs, tasks, lr);
    int ev;
    launch_gemm<Fc1Dgrad<T, F1D_BM, F1D_BN>, F1D_BM, F1D_BN>(ctx, {drecs, d}, L, OP_F1D, dtab);
    launch_gemm<Fc1Wgrad<T, F1W_BM, F1W_BN>, F1W_BM, F1W_BN>(ctx, {drecs, d, lr}, L, OP_F1W, dtab);
    launch_gemm<Conv2Dgrad<T, C2D_BM, C2D_BN>, C2D_BM, C2D_BN>(ctx, {drecs, d}, L, OP_C2D, dtab);
    launch_gemm<Conv2Wgrad<T, C2W_BM, C2W_BN>, C2W_BM, C2W_BN>(ctx, {drecs, d}, L, OP_C2W, dtab);
    ReduceArgs r2{drecs, B_WSP, m.c2, 25 * m.c1, d.w2, d.b2, d.HW2(), lr, 0, -1};
    ev = op_begin(ctx, OP_C2R, OP_C2R);
    k_reduce_update<<<L.grid[OP_C2R], kReduceBlock, 0, ctx->cur>>>(r2, tasks, dtab + L.prefix_off[OP_C2R],
                                                                       L.ntask);
    op_end(ctx, ev);
    launch_gemm<Conv1Wgrad<T, C1W_BM, C1W_BN>, C1W_BM, C1W_BN>(ctx, {drecs, d}, L, OP_C1W, dtab);
    ReduceArgs r1{drecs, B_WSP, m.c1, 25 * d.C, d.w1, d.b1, d.HW(), lr, 0, -1};
    ev = op_begin(ctx, OP_C1R, OP_C1R);
    k_reduce_update<<<L.grid[OP_C1R], kReduceBlock, 0, ctx->cur>>>(r1, tasks, dtab + L.prefix_off[OP_C1R],
                                                                       L.ntask);
    op_end(ctx, ev);
  } else if (m.arch == PROTEA_MODEL_MLP) {
    const MlpDims d = mlp_dims(m);
    {
      const size_t smem = (16 * 784 + 256) * 4 + 64 * 784;
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(k_mlp_fc1_fwd<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
      }
      const int ev = op_begin(ctx, OP_MF, OP_MF);
      k_mlp_fc1_fwd<T><<<dim3(L.ntask, 4), kMlpFwdThreads, smem, ctx->cur>>>(drecs, tasks, d);
      op_end(ctx, ev);
    }
    if (ctx->eval_mode) {
      launch_eval<T>(ctx, L, drecs, tasks, B_H1, 64, 1, m.layers[1], m.classes);
      return;
    }
    HeadArgs ha{drecs, B_H1, B_DZ1, 64, m.classes, d.w2, d.b2, d.b1, lr};
    const int ev = op_begin(ctx, OP_MHEAD, OP_MHEAD);
    k_head<T><<<L.ntask, kHeadThreads, 0, ctx->cur>>>(ha, tasks);
    op_end(ctx, ev);
    launch_gemm<MlpFc1Wgrad<T, MW_BM, MW_BN>, MW_BM, MW_BN>(ctx, {drecs, d, lr}, L, OP_MW, dtab);
  }
}

int grid_for(int64_t n, int threads, int cap = 148 * 8) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, cap));
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {
uint64_t protea_plan_hash(const protea_client* clients, size_t n, const protea_assignment* plan) {
  uint64_t h = 1469598103934665603ull;  // FNV-1a 64
  auto mix = [&h](const void* p, size_t bytes) {
    const uint8_t* b = static_cast<const uint8_t*>(p);
    for (size_t i = 0; i < bytes; ++i) {
      h ^= b[i];
      h *= 1099511628211ull;
    }
  };
  mix(&n, sizeof(n));
  for (size_t i = 0; clients && i < n; ++i) {
    mix(&clients[i].client_id, 8);
    mix(&clients[i].model_id, 4);
    mix(&clients[i].batch, 4);
    mix(&clients[i].epochs, 4);
  }
  for (size_t i = 0; plan && i < n; ++i) {
    mix(&plan[i].client_id, 8);
    mix(&plan[i].gpu, 4);
    mix(&plan[i].q1024, 4);
    mix(&plan[i].offset, 8);
    mix(&plan[i].slot, 8);
    mix(&plan[i].admit, 8);
    mix(&plan[i].release, 8);
  }
  return h;
}

// Debug cycle counters of instrumented kernels (built with -DPROTEA_DBG=1); not part of the public ABI.
int protea_debug_counters(uint64_t* out, int reset) {
  if (cudaMemcpyFromSymbol(out, protea::g_dbg, 64 * sizeof(uint64_t)) != cudaSuccess) return -1;
  if (reset) {
    const uint64_t z[64] = {};
    cudaMemcpyToSymbol(protea::g_dbg, z, sizeof(z));
  }
  return 0;
}


const char* protea_last_error(const protea_ctx* ctx) {
  if (ctx) return ctx->err.c_str();
  std::lock_guard<std::mutex> lk(g_err_mu);
  return g_err.c_str();
}

protea_status protea_init(const protea_init_opts* opts, protea_ctx** out) {
  if (!opts || !out) {
    set_global_error("protea_init: null argument");
    return PROTEA_ERR_INVALID;
  }
  if (opts->world < 1 || opts->rank < 0 || opts->rank >= opts->world ||
      !opts->arena || opts->arena_bytes == 0 ||
      (opts->precision != PROTEA_PREC_FP32 && opts->precision != PROTEA_PREC_BF16)) {
    set_global_error("protea_init: invalid rank/world/nccl_id/arena/precision");
    return PROTEA_ERR_INVALID;
  }
  std::unique_ptr<protea_ctx> c(new protea_ctx());
  c->device = opts->device;
  c->rank = opts->rank;
  c->world = opts->world;
  c->precision = opts->precision;
  c->stream = (cudaStream_t)opts->stream;
  c->arena = (uint8_t*)opts->arena;
  c->arena_bytes = opts->arena_bytes;
  protea_ctx* ctx = c.get();
  cudaError_t e = cudaSetDevice(opts->device);
  if (e != cudaSuccess) {
    set_global_error(std::string("protea_init: cudaSetDevice: ") + cudaGetErrorString(e));
    return PROTEA_ERR_CUDA;
  }
  ctx->cur = ctx->stream;
  {
    int nsm = 0;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, opts->device) == cudaSuccess && nsm > 0)
      g_num_sms = nsm;
  }
  int prio_least = 0, prio_greatest = 0;
  cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest);
  if (const char* ov = std::getenv("PROTEA_OVERLAP_ROWS")) ctx->overlap_rows = std::atoll(ov);
  if (const char* pd = std::getenv("PROTEA_PDL")) ctx->pdl = std::atoi(pd) != 0;
  if (const char* fs = std::getenv("PROTEA_F1W_SIDE_SMEM")) ctx->f1w_side_smem = std::max(0, std::min(220 * 1024, std::atoi(fs)));
  if (const char* dc = std::getenv("PROTEA_DEFER_C2R")) ctx->defer_c2r = std::atoi(dc) != 0;
  if (const char* ro = std::getenv("PROTEA_R8_OVERLAP")) ctx->r8_overlap = std::atoi(ro) != 0;
  g_r8_halo = 15;  // (process-wide: every context re-reads it, so an earlier context's setting does not leak)
  if (const char* rh = std::getenv("PROTEA_R8_HALO")) g_r8_halo = std::atoi(rh) & 15;
  if (const char* rr = std::getenv("PROTEA_R8_OVERLAP_ROWS")) ctx->r8_overlap_rows = std::atoll(rr);
  if (const char* ln = std::getenv("PROTEA_LANES")) ctx->lanes = std::max(1, std::min(4, std::atoi(ln)));
  if (cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, prio_least) != cudaSuccess ||
      cudaStreamCreateWithPriority(&ctx->hi, cudaStreamNonBlocking, prio_greatest) != cudaSuccess ||
      cudaStreamCreateWithPriority(&ctx->wstream, cudaStreamNonBlocking, prio_greatest) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming) != cudaSuccess) {
    set_global_error("protea_init: stream/event creation failed");
    return PROTEA_ERR_CUDA;
  }
  if (cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess) {
    set_global_error("protea_init: cudaEventCreate failed");
    return PROTEA_ERR_CUDA;
  }
  if (opts->nccl_id) {  // also world == 1: a one-rank communicator runs the same exchange path
    ncclUniqueId id;
    std::memcpy(&id, opts->nccl_id, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&ctx->comm, opts->world, id, opts->rank);
    if (r != ncclSuccess) {
      set_global_error(std::string("protea_init: ncclCommInitRank: ") + ncclGetErrorString(r));
      return PROTEA_ERR_NCCL;
    }
  }
  *out = c.release();
  return PROTEA_OK;
}

void protea_finalize(protea_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (auto* mp : {&ctx->shards, &ctx->val_shards})
    for (auto& kv : *mp) {
      cudaFree(kv.second.x);
      cudaFree(kv.second.y);
    }
  ctx->gin.release();
  ctx->gout.release();
  ctx->acc.release();
  ctx->gath.release();
  ctx->flag.release();
  ctx->regions.release();
  ctx->hwm.release();
  ctx->recs.release();
  ctx->tab.release();
  ctx->ev_recs.release();
  ctx->ev_tab.release();
  ctx->ev_ws.release();
  ctx->ev_loss.release();
  ctx->ev_ok.release();
  ctx->ptrs.release();
  ctx->wts.release();
  ctx->wq.release();
  for (auto e : ctx->evpool) cudaEventDestroy(e);
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
  }
  if (ctx->hi) {
    cudaStreamSynchronize(ctx->hi);
    cudaStreamDestroy(ctx->hi);
  }
  if (ctx->wstream) {
    cudaStreamSynchronize(ctx->wstream);
    cudaStreamDestroy(ctx->wstream);
  }
  for (auto e : ctx->r8ev)
    if (e) cudaEventDestroy(e);
  for (auto e : ctx->gjoin) cudaEventDestroy(e);
  for (auto sgs : ctx->gstream) {
    cudaStreamSynchronize(sgs);
    cudaStreamDestroy(sgs);
  }
  for (auto e : ctx->gdone) cudaEventDestroy(e);
  if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
  if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  delete ctx;
}

protea_status protea_register_model(protea_ctx* ctx, const protea_model_desc* desc, int32_t* model_id,
                                    uint64_t* n_params) {
  if (!ctx) return PROTEA_ERR_INVALID;
  if (!desc || !model_id || !n_params) return fail(ctx, PROTEA_ERR_INVALID, "register_model: null argument");
  Group g;
  std::string err;
  if (!make_model(*desc, &g.m, &err)) return fail(ctx, PROTEA_ERR_INVALID, "register_model: " + err);
  // every shard of a context is read with one input size D (register_shards copies n * D bytes)
  if (!ctx->groups.empty() && g.m.in_dim() != ctx->groups[0].m.in_dim())
    return fail(ctx, PROTEA_ERR_INVALID, "register_model: input size " + std::to_string(g.m.in_dim()) +
                                             " differs from the registered models' " +
                                             std::to_string(ctx->groups[0].m.in_dim()) + " (one input size per context)");
  g.offset = 0;
  for (auto& x : ctx->groups) g.offset += x.m.P;
  ctx->groups.push_back(g);
  *model_id = (int32_t)ctx->groups.size() - 1;
  *n_params = (uint64_t)g.m.P;
  return PROTEA_OK;
}

static protea_status register_into(protea_ctx* ctx, std::map<int64_t, ShardDev>& dst, const protea_shard* shards,
                                   size_t n) {
  if (!ctx) return PROTEA_ERR_INVALID;
  if (!shards || n == 0) return fail(ctx, PROTEA_ERR_INVALID, "register_shards: null or empty");
  for (size_t i = 0; i < n; ++i)
    if (shards[i].n <= 0 || !shards[i].x || !shards[i].y)
      return fail(ctx, PROTEA_ERR_INVALID,
                  "register_shards: client " + std::to_string(shards[i].client_id) + " has n <= 0 or null data");
  // all shards of a context share one input size D (taken from the first registered model, else from
  // the caller's bytes per example: x holds n * D bytes; D is inferred per call from the models).
  if (ctx->groups.empty()) return fail(ctx, PROTEA_ERR_INVALID, "register_shards: register a model first");
  const int64_t D = ctx->groups[0].m.in_dim();
  CK(cudaSetDevice(ctx->device));
  for (size_t i = 0; i < n; ++i) {
    const protea_shard& s = shards[i];
    auto it = dst.find(s.client_id);
    ShardDev d;
    if (it != dst.end() && it->second.n == s.n) {
      d = it->second;  // same size: refresh the device copy in place
    } else {
      if (it != dst.end()) {
        cudaFree(it->second.x);
        cudaFree(it->second.y);
        dst.erase(it);
      }
      d.n = s.n;
      d.x = nullptr;
      d.y = nullptr;
      CK(cudaMalloc(&d.x, (size_t)s.n * D));
      CK(cudaMalloc(&d.y, (size_t)s.n * 4));
    }
    d.ymin = *std::min_element(s.y, s.y + s.n);
    d.ymax = *std::max_element(s.y, s.y + s.n);
    CK(cudaMemcpyAsync(d.x, s.x, (size_t)s.n * D, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(d.y, s.y, (size_t)s.n * 4, cudaMemcpyHostToDevice, ctx->stream));
    dst[s.client_id] = d;
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return PROTEA_OK;
}

protea_status protea_register_shards(protea_ctx* ctx, const protea_shard* shards, size_t n) {
  if (!ctx) return PROTEA_ERR_INVALID;
  return register_into(ctx, ctx->shards, shards, n);
}

protea_status protea_register_val_shards(protea_ctx* ctx, const protea_shard* shards, size_t n) {
  if (!ctx) return PROTEA_ERR_INVALID;
  return register_into(ctx, ctx->val_shards, shards, n);
}

protea_status protea_client_footprint(const protea_model_desc* desc, int64_t n, int32_t batch, int32_t epochs,
                                      int32_t precision, uint64_t* peak_bytes, uint64_t* steps, uint64_t* flops) {
  if (!desc || !peak_bytes || !steps || !flops || n <= 0 || batch <= 0 || epochs <= 0 ||
      (precision != PROTEA_PREC_FP32 && precision != PROTEA_PREC_BF16)) {
    set_global_error("client_footprint: invalid argument");
    return PROTEA_ERR_INVALID;
  }
  ModelDims m;
  std::string err;
  if (!make_model(*desc, &m, &err)) {
    set_global_error("client_footprint: " + err);
    return PROTEA_ERR_INVALID;
  }
  *peak_bytes = client_hwm(m, batch, n, epochs, precision == PROTEA_PREC_FP32 ? 4 : 2);
  *steps = (uint64_t)epochs * ceil_div((uint64_t)n, (uint64_t)batch);
  *flops = (uint64_t)epochs * (uint64_t)n * flops_per_sample(m);
  return PROTEA_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// round execution (shared by protea_run_round and the profiler's probe)
// ---------------------------------------------------------------------------
namespace {

struct RunClient {
  int64_t id;
  int group;
  int64_t n;
  int B, E, nb;
  uint64_t S, admit, release;
  uint64_t offset;
  uint64_t slot = 0;  // planned slot bytes (observe_hwm poisons / scans [offset, offset + slot))
  // micro-clients (batches above kMicroRows rows, common.h): execute() expands such a client into
  // micro-clients micro = 0..nmicro-1, each holding rows [micro * kMicroRows, +cap) of every batch
  int orig = -1;      // index of the client in execute()'s input
  int micro = 0, nmicro = 1;
  int cap = 0;        // rows this (micro-)client's slot holds: min(B, n) or its share of it
  uint64_t mw_off = 0;  // micro 0: arena offset of the merge weights
  int rec = -1;
  int lane = 0;  // lock-step lane within the model group (PROTEA_LANES)
};

// Rows of (micro-)client c's batch in lock-step iteration t (0: the micro has no rows in this batch).
int micro_rows(const RunClient& c, uint64_t t) {
  const int64_t j = (int64_t)((t - c.admit) % c.nb);
  const int64_t rb = std::min<int64_t>(c.B, c.n - j * c.B);
  return (int)std::max<int64_t>(0, std::min<int64_t>(c.cap, rb - (int64_t)c.micro * kMicroRows));
}

// Verification / observation extras of one execute() call.
struct ExecExtras {
  bool observe = false;             // poison each slot at admission, scan it at release -> ctx->hwm[rec]
  std::map<int64_t, uint8_t*> trace;  // client id -> device buffer of (S_k + 1) slot snapshots
  bool eval = false;                  // evaluate round: forward + classifier head, no update, no merge
  const std::map<int64_t, ShardDev>* shards = nullptr;  // data to read (default: the training shards)
  std::vector<double>* stats_out = nullptr;  // eval: per input client (loss sum, correct) from stats[0], [2]
};

// Validates and executes the lock-step schedule of `rc` (this rank's clients,
// ascending id) inside the arena.  wg: device concatenated global weights;
// acc: device fp64 accumulator (zeroed by caller) or nullptr (probe mode:
// no FedAvg terms).  Returns iterations run.
protea_status execute(protea_ctx* ctx, std::vector<RunClient>& rc_in, const float* wg, double* acc, float lr,
                      uint32_t seed, uint32_t round, int shuffle, uint64_t* iters_out, double* loss_dev,
                      const ExecExtras* xx = nullptr) {
  const int e = ctx->precision == PROTEA_PREC_FP32 ? 4 : 2;
  const bool tc_mode = e == 2;  // bf16 mode: tensor-core GEMMs for the CNN
  const int G = (int)ctx->groups.size();
  struct EvalFlag {  // ctx->eval_mode for the duration of this call (every return path)
    protea_ctx* c;
    EvalFlag(protea_ctx* c_, bool on) : c(c_) { c->eval_mode = on; }
    ~EvalFlag() { c->eval_mode = false; }
  } eval_flag(ctx, xx && xx->eval);
  // ---- micro-clients: a client whose batch holds more than kMicroRows rows becomes nmicro micro-clients
  // (slots back to back inside its slot, then the merge weights); results are reported per input client
  std::vector<RunClient> rc;
  bool have_micro = false;
  for (size_t i = 0; i < rc_in.size(); ++i) {
    const RunClient& c = rc_in[i];
    const ModelDims& m = ctx->groups[c.group].m;
    const int64_t beff = std::min<int64_t>(c.B, c.n);
    const int M = micro_count(c.B, c.n);
    uint64_t off = c.offset;
    for (int k = 0; k < M; ++k) {
      RunClient x = c;
      x.orig = (int)i;
      x.micro = k;
      x.nmicro = M;
      x.cap = (int)std::min<int64_t>(M == 1 ? beff : kMicroRows, beff - (int64_t)k * kMicroRows);
      x.offset = off;
      x.slot = k == 0 ? c.slot : 0;  // observe_hwm: micro 0's region is the whole client slot
      off += slot_layout(m, x.cap, c.n, c.E, e).total;
      rc.push_back(x);
    }
    if (M > 1) {
      rc[rc.size() - M].mw_off = off;
      have_micro = true;
    }
  }
  // ---- device records
  std::vector<ClientRec> recs(rc.size());
  std::vector<int64_t> gacc_off(G, 0);
  for (int g = 1; g < G; ++g) gacc_off[g] = gacc_off[g - 1] + ctx->groups[g - 1].m.P;
  for (size_t i = 0; i < rc.size(); ++i) {
    RunClient& c = rc[i];
    c.rec = (int)i;
    const Group& gr = ctx->groups[c.group];
    const SlotLayout L = slot_layout(gr.m, c.cap, c.n, c.E, e);
    ClientRec& r = recs[i];
    std::memset(&r, 0, sizeof(r));
    uint8_t* base = ctx->arena + c.offset;
    for (int b = 0; b < B_COUNT; ++b) r.buf[b] = L.used[b] ? base + L.off[b] : nullptr;
    r.params = (float*)r.buf[B_PARAMS];
    r.perm = (int32_t*)r.buf[B_PERM];
    r.stats = (float*)r.buf[B_STATS];
    const ShardDev& sd = (xx && xx->shards ? *const_cast<std::map<int64_t, ShardDev>*>(xx->shards) : ctx->shards)[c.id];
    r.x = sd.x;
    r.y = sd.y;
    r.wg = wg + gr.offset;
    r.acc = acc ? acc + gacc_off[c.group] : nullptr;
    r.n = (int32_t)c.n;
    r.B = c.cap;  // rows a batch can hold here: the slot's per-row buffer capacity
    r.mw = c.mw_off ? (float*)(ctx->arena + c.mw_off) : nullptr;
    if (tc_mode && gr.m.arch == PROTEA_MODEL_CNN && gr.m.H == 32) {  // fc1's W as split planes (device.cuh)
      r.sp_off = gr.m.layers[2].off_w;
      r.sp_len = (int64_t)gr.m.layers[2].cout * gr.m.layers[2].K();
      r.sp_k = gr.m.layers[2].K();
    }
    r.E = c.E;
    r.nb = c.nb;
    r.id = c.id;
    r.P = gr.m.P;
    r.c1 = gr.m.c1;
  }
  // ---- observed high-water marks (poisoned slots) and traced clients
  const bool observe = xx && xx->observe;
  std::vector<uint8_t*> trace_of(rc.size(), nullptr);
  std::vector<uint64_t> trace_bytes(rc.size(), 0);  // a snapshot = the whole slot layout (params first)
  if (xx)
    for (size_t i = 0; i < rc.size(); ++i) {
      auto it = xx->trace.find(rc[i].id);
      if (it != xx->trace.end() && rc[i].micro == 0) {  // the whole client slot (all micro slots)
        trace_of[i] = it->second;
        trace_bytes[i] = client_hwm(ctx->groups[rc[i].group].m, rc[i].B, rc[i].n, rc[i].E, e);
      }
    }
  uint64_t max_slot = 0;
  if (observe) {
    std::vector<uint64_t> reg(3 * rc.size());
    for (size_t i = 0; i < rc.size(); ++i) {
      reg[3 * i] = rc[i].offset;
      reg[3 * i + 1] = rc[i].slot;
      reg[3 * i + 2] = (uint64_t)rc[i].orig;  // observed mark reported per input client
      max_slot = std::max(max_slot, rc[i].slot);
    }
    CK(ctx->regions.reserve(reg.size()));
    CK(ctx->hwm.reserve(rc_in.size()));
    CK(cudaMemcpyAsync(ctx->regions.p, reg.data(), reg.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(ctx->hwm.p, 0, rc_in.size() * 8, ctx->stream));
  }
  // ---- K9 per-client SM-time counters
  CK(ctx->smns.reserve(std::max<size_t>(rc_in.size(), 1)));
  CK(cudaMemsetAsync(ctx->smns.p, 0, std::max<size_t>(rc_in.size(), 1) * 8, ctx->stream));
  for (size_t i = 0; i < rc.size(); ++i) recs[i].sm_ns = ctx->smns.p + rc[i].orig;  // micros add up
  // ---- TMA tensor maps (bf16 CNN clients)
  if (tc_mode) {
    std::vector<CUtensorMap> maps;
    std::vector<int> owner;
    for (size_t i = 0; i < rc.size(); ++i) {
      const ModelDims& m = ctx->groups[rc[i].group].m;
      const bool r8 = m.arch == PROTEA_MODEL_RESNET8 && g_r8_halo != 0;
      if (!(m.arch == PROTEA_MODEL_CNN && m.H == 32) && !r8) continue;
      auto key = std::make_tuple(rc[i].offset, rc[i].cap, rc[i].E, rc[i].n, rc[i].group);
      auto it = ctx->tmap_cache.find(key);
      if (it == ctx->tmap_cache.end()) {
        std::array<CUtensorMap, kTmapSlots> a;
        std::memset(a.data(), 0, sizeof(a));
        if (!(r8 ? build_r8_tmaps(m, recs[i], recs[i].B, a.data()) : build_cnn_tmaps(m, recs[i], recs[i].B, a.data())))
          return fail(ctx, PROTEA_ERR_CUDA, "run_round: cuTensorMapEncodeTiled failed for client " +
                                               std::to_string(rc[i].id));
        it = ctx->tmap_cache.emplace(key, a).first;
      }
      owner.push_back((int)i);
      maps.insert(maps.end(), it->second.begin(), it->second.end());
    }
    if (!maps.empty()) {
      CK(ctx->tmaps.reserve(maps.size()));
      CK(cudaMemcpyAsync(ctx->tmaps.p, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice,
                         ctx->stream));
      for (size_t k = 0; k < owner.size(); ++k) recs[owner[k]].tmaps = ctx->tmaps.p + k * kTmapSlots;
    }
  }
  // ---- lock-step lanes: within each (group, batch size) class the clients alternate between lanes, so
  // every lane gets the same mix of step counts; each lane is an independent chain on its own stream.
  // Micro-clients run in one extra lane per group (their SGD steps use lr * kMicroLrScale)
  const int NL0 = tc_mode ? ctx->lanes : 1;
  const int NL = NL0 + (have_micro ? 1 : 0);
  {
    std::map<std::pair<int, int>, int> seen_class;
    for (auto& c : rc) c.lane = c.nmicro > 1 ? NL0 : (NL0 > 1 ? seen_class[{c.group, c.B}]++ % NL0 : 0);
  }
  // ---- schedule tables
  uint64_t T = 0;
  for (auto& c : rc) T = std::max(T, c.release);
  std::vector<int32_t> tab;
  std::vector<Launch> launches;
  std::vector<std::pair<int64_t, int>> admits(T + 1, {-1, 0}), rels;  // per-iteration (offset, count)
  std::vector<std::vector<std::pair<int64_t, int>>> rel_by_group(T + 1, std::vector<std::pair<int64_t, int>>(G, {-1, 0}));
  std::vector<std::vector<int>> launch_idx(T);
  struct Merge {
    int64_t off;
    int rec0, R;
  };
  std::vector<std::vector<Merge>> merges(T);
  for (uint64_t t = 0; t < T; ++t) {
    // admissions at t (ascending id)
    std::vector<int> adm;
    for (auto& c : rc)
      if (c.admit == t) adm.push_back(c.rec);
    if (!adm.empty()) {
      admits[t] = {(int64_t)tab.size(), (int)adm.size()};
      tab.insert(tab.end(), adm.begin(), adm.end());
    }
    for (int v = 0; v < G * NL; ++v) {
      const int g = v / NL, lane = v % NL;
      const ModelDims& m = ctx->groups[g].m;
      std::vector<const RunClient*> act;
      for (auto& c : rc)
        if (c.group == g && c.lane == lane && c.admit <= t && t < c.release && micro_rows(c, t) > 0)
          act.push_back(&c);
      if (!act.empty()) {
        Launch L;
        std::memset(&L, 0, sizeof(L));
        L.group = g;
        L.vg = v;
        L.ntask = (int)act.size();
        while (tab.size() % 4) tab.push_back(0);
        L.task_off = (int64_t)tab.size();
        std::vector<int> rows(act.size());
        for (size_t i = 0; i < act.size(); ++i) {
          const RunClient& c = *act[i];
          const int s = (int)(t - c.admit), ep = s / c.nb, j = s % c.nb;
          rows[i] = micro_rows(c, t);
          L.max_rows = std::max(L.max_rows, rows[i]);
          tab.push_back(c.rec);
          tab.push_back((int32_t)std::min<int64_t>(c.B, c.n - (int64_t)j * c.B));  // |beta| of the whole batch
          tab.push_back(rows[i]);
          tab.push_back((int32_t)((int64_t)ep * c.n + (int64_t)j * c.B + (int64_t)c.micro * kMicroRows));
        }
        // width-1 conv2 wgrad: when the iteration has few splits (the tail), each split's 7 M tiles become
        // 7 work items (no extra partials: disjoint outputs), otherwise one item covers all 7 tiles
        L.c2w_groups = 1;
        if (tc_mode && m.arch == PROTEA_MODEL_CNN && m.width_q == 4 && m.H == 32) {
          int64_t nsplit = 0;
          for (int r : rows) nsplit += cdiv(r * 256, kWgradChunkPx);
          if (nsplit < 2 * g_num_sms) L.c2w_groups = 7;
        }
        for (int op : ops_of(m, tc_mode)) {
          L.prefix_off[op] = (int64_t)tab.size();
          int acc_t = 0;
          for (size_t i = 0; i < act.size(); ++i) {
            tab.push_back(acc_t);
            acc_t += tiles(m, op, rows[i], tc_mode) * (op == OP_C2W ? L.c2w_groups : 1);
            uint64_t fl, by;
            op_work(m, op, (uint64_t)rows[i], (uint64_t)e, &fl, &by);
            ctx->op_flops[op_class(op)] += fl;
            ctx->op_bytes[op_class(op)] += by;
            L.fl[op] += fl;
            L.by[op] += by;
          }
          tab.push_back(acc_t);
          L.grid[op] = acc_t;
        }
        launch_idx[t].push_back((int)launches.size());
        launches.push_back(L);
      }
    }
    // micro-client merges after iteration t: [M recs][M rows] per client whose batch is split
    for (auto& c : rc)
      if (c.nmicro > 1 && c.micro == 0 && c.admit <= t && t < c.release) {
        int R = 0;
        const int64_t off = (int64_t)tab.size();
        for (int k = 0; k < c.nmicro; ++k) tab.push_back(c.rec + k);
        for (int k = 0; k < c.nmicro; ++k) {
          const int r = micro_rows(rc[c.rec + k], t);
          tab.push_back(r);
          R += r;
        }
        merges[t].push_back({off, c.rec, R});
      }
    for (int g = 0; g < G; ++g) {
      // releases after iteration t (client finished its last step), all lanes, ascending id
      std::vector<int> rel;
      for (auto& c : rc)
        if (c.group == g && c.release == t + 1 && c.micro == 0) rel.push_back(c.rec);
      if (!rel.empty()) {
        rel_by_group[t][g] = {(int64_t)tab.size(), (int)rel.size()};
        tab.insert(tab.end(), rel.begin(), rel.end());
      }
    }
  }
  CK(ctx->recs.reserve(recs.size()));
  CK(ctx->tab.reserve(tab.size()));
  CK(cudaMemcpyAsync(ctx->recs.p, recs.data(), recs.size() * sizeof(ClientRec), cudaMemcpyHostToDevice, ctx->stream));
  if (!tab.empty())
    CK(cudaMemcpyAsync(ctx->tab.p, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
  const ClientRec* drecs = ctx->recs.p;
  const int32_t* dtab = ctx->tab.p;
  int maxE = 1;
  for (auto& c : rc) maxE = std::max(maxE, c.E);
  // the iterations run on the high-priority stream (forked from / joined into the caller's stream)
  while ((int)ctx->gjoin.size() < G) {
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    ctx->gjoin.push_back(ev);
  }
  ctx->gpending.assign(G, 0);
  // group g > 0 runs on its own stream (same priority as hi); admissions join every group first
  const int V = G * NL;
  while ((int)ctx->gstream.size() < V) {
    int lo = 0, hi_p = 0;
    cudaStream_t sgs;
    cudaEvent_t ev;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi_p));
    CK(cudaStreamCreateWithPriority(&sgs, cudaStreamNonBlocking, hi_p));
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    ctx->gstream.push_back(sgs);
    ctx->gdone.push_back(ev);
  }
  std::vector<cudaStream_t> gs(V, ctx->hi);
  for (int v = 1; v < V; ++v) gs[v] = ctx->serialize ? ctx->hi : ctx->gstream[v];  // serialize: one stream
  ctx->spin_cap = std::max(1, g_num_sms / (ctx->serialize ? 1 : NL));  // one spin-waiting wgrad per lane at a time
  ctx->single_chain = V == 1;
  CK(cudaEventRecord(ctx->fork_ev, ctx->stream));
  CK(cudaStreamWaitEvent(ctx->hi, ctx->fork_ev, 0));
  ctx->cur = ctx->hi;
  auto join_groups_into_hi = [&]() {  // hi waits for every other lane stream
    for (int v = 1; v < V; ++v) {
      cudaEventRecord(ctx->gdone[v], gs[v]);
      cudaStreamWaitEvent(ctx->hi, ctx->gdone[v], 0);
    }
  };
  auto fork_groups_from_hi = [&]() {  // every other lane stream waits for hi
    if (V > 1) {
      cudaEventRecord(ctx->gdone[0], ctx->hi);
      for (int v = 1; v < V; ++v) cudaStreamWaitEvent(gs[v], ctx->gdone[0], 0);
    }
  };
  fork_groups_from_hi();
  std::vector<int64_t> iter_rows(T, 0);
  for (auto& c : rc)
    for (uint64_t t = c.admit; t < c.release; ++t) {
      iter_rows[t] += micro_rows(c, t);
    }
  NvtxRange nv_iters("protea: lock-step iterations");
  for (uint64_t t = 0; t < T; ++t) {
    char nv_name[48];
    std::snprintf(nv_name, sizeof(nv_name), "iteration %llu (%lld rows)", (unsigned long long)t,
                  (long long)iter_rows[t]);
    nvtxRangePushA(nv_name);
    struct NvPop { ~NvPop() { nvtxRangePop(); } } nv_pop;
    // (several groups already overlap each other: no side-stream deferral then)
    ctx->overlap_now = tc_mode && !ctx->serialize && V == 1 && iter_rows[t] <= ctx->overlap_rows;
    ctx->rows_now = iter_rows[t];
    if (admits[t].second > 0) {
      // an admitted client may reuse a slot released by any group: every group's earlier work first
      ctx->cur = ctx->hi;
      if (t > 0) join_groups_into_hi();
      const int* ids = dtab + admits[t].first;
      int64_t maxP = 0, maxn = 0;
      for (auto& c : rc)
        if (c.admit == t) {
          maxP = std::max<int64_t>(maxP, ctx->groups[c.group].m.P);
          maxn = std::max<int64_t>(maxn, c.n);
        }
      for (auto& c : rc)
        if (c.admit == t) ctx->op_bytes[PROTEA_OPC_ADMIT] += 8 * (uint64_t)ctx->groups[c.group].m.P + 4 * (uint64_t)c.E * c.n;
      if (observe) {
        k_fill_poison<<<dim3(grid_for((int64_t)(max_slot / 16), 256, 4 * g_num_sms), admits[t].second), 256, 0,
                        ctx->cur>>>(ctx->arena, ctx->regions.p, ids);
        ctx->launches++;
      }
      int ev = op_begin(ctx, PROTEA_OPC_ADMIT);
      k_admit_params<<<dim3(grid_for(maxP / 4 + 1, 256, 64), admits[t].second), 256, 0, ctx->cur>>>(drecs, ids);
      op_end(ctx, ev);
      ev = op_begin(ctx, PROTEA_OPC_ADMIT);
      k_admit_perm<<<dim3(cdiv((int)maxn, kPermThreads), admits[t].second, maxE), kPermThreads, 0, ctx->cur>>>(
          drecs, ids, seed, round, shuffle);
      op_end(ctx, ev);
      for (auto& c : rc)  // snapshot 0 of a traced client: the weights it starts from
        if (c.admit == t && trace_of[c.rec])
          CK(cudaMemcpyAsync(trace_of[c.rec], recs[c.rec].params, trace_bytes[c.rec], cudaMemcpyDeviceToDevice,
                             ctx->cur));
      fork_groups_from_hi();
    }
    for (int li : launch_idx[t]) {
      const Launch& L = launches[li];
      const ModelDims& m = ctx->groups[L.group].m;
      ctx->cur = gs[L.vg];
      ctx->cur_fl = L.fl;
      ctx->cur_by = L.by;
      // micro-client lane: SGD steps scaled by the exact power of two kMicroLrScale (k_micro_merge)
      const float lr_l = have_micro && L.vg % NL == NL0 ? lr * kMicroLrScale : lr;
      if (e == 4)
        launch_step<float>(ctx, m, L, drecs, dtab, lr_l);
      else if (m.arch == PROTEA_MODEL_CNN && m.H == 32)
        launch_step_tc(ctx, m, L, drecs, dtab, lr_l);
      else
        launch_step<__nv_bfloat16>(ctx, m, L, drecs, dtab, lr_l);
    }
    for (const Merge& mg : (ctx->eval_mode ? std::vector<Merge>() : merges[t])) {  // w' = w + sum_m (b_m / R)(w_m - w) / scale; reload every micro
      const RunClient& c0 = rc[mg.rec0];
      ctx->cur = gs[c0.group * NL + c0.lane];
      join_group(ctx, c0.group);
      const int64_t P = ctx->groups[c0.group].m.P;
      k_micro_merge<<<grid_for(P, 256), 256, 0, ctx->cur>>>(drecs, dtab + mg.off, c0.nmicro, mg.R);
      k_micro_bcast<<<dim3(grid_for(P, 256, 64), c0.nmicro), 256, 0, ctx->cur>>>(drecs, dtab + mg.off);
      ctx->launches += 2;
    }
    for (auto& c : rc)  // snapshot s = t - admit + 1 of a traced client (after its deferred work)
      if (trace_of[c.rec] && c.admit <= t && t < c.release) {
        ctx->cur = gs[c.group * NL + c.lane];
        join_group(ctx, c.group);
        CK(cudaMemcpyAsync(trace_of[c.rec] + (t - c.admit + 1) * trace_bytes[c.rec], recs[c.rec].params,
                           trace_bytes[c.rec], cudaMemcpyDeviceToDevice, ctx->cur));
      }
    if (acc || observe)
      for (int g = 0; g < G; ++g)
        if (rel_by_group[t][g].second > 0) {
          const int64_t P = ctx->groups[g].m.P;
          ctx->cur = gs[g * NL];
          for (int l = 1; l < NL; ++l) {  // the group's other lanes finished iteration t first
            cudaEventRecord(ctx->gdone[g * NL + l], gs[g * NL + l]);
            cudaStreamWaitEvent(ctx->cur, ctx->gdone[g * NL + l], 0);
          }
          join_group(ctx, g);  // the released clients' last fc1 wgrad
          if (acc) {
            ctx->op_bytes[PROTEA_OPC_FEDAVG] += (uint64_t)P * (20 + 4 * rel_by_group[t][g].second);
            const int ev = op_begin(ctx, PROTEA_OPC_FEDAVG);
            k_release_acc<<<grid_for(P, 256), 256, 0, ctx->cur>>>(drecs, dtab + rel_by_group[t][g].first,
                                                                   rel_by_group[t][g].second, P, loss_dev + g);
            op_end(ctx, ev);
          }
          if (observe) {  // the released clients' slots: highest byte touched during their whole lifetime
            k_scan_poison<<<dim3(grid_for((int64_t)(max_slot / 16), 256, 2 * g_num_sms), rel_by_group[t][g].second),
                            256, 0, ctx->cur>>>(ctx->arena, ctx->regions.p, dtab + rel_by_group[t][g].first,
                                                ctx->hwm.p);
            ctx->launches++;
          }
        }
  }
  for (int g = 0; g < G; ++g) {
    ctx->cur = gs[g * NL];
    join_group(ctx, g);
  }
  ctx->cur = ctx->hi;
  join_groups_into_hi();
  ctx->overlap_now = false;
  ctx->cur_fl = ctx->cur_by = nullptr;
  CK(cudaEventRecord(ctx->join_ev, ctx->hi));
  CK(cudaStreamWaitEvent(ctx->stream, ctx->join_ev, 0));
  ctx->cur = ctx->stream;
  CK(cudaGetLastError());
  if (iters_out) *iters_out = T;
  if (xx && xx->stats_out) {  // evaluate round: per input client (loss sum, correct), micro-clients summed
    std::vector<float> st(3 * rc.size());
    for (size_t i = 0; i < rc.size(); ++i)
      CK(cudaMemcpyAsync(&st[3 * i], recs[i].stats, 12, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    xx->stats_out->assign(2 * rc_in.size(), 0.0);
    for (size_t i = 0; i < rc.size(); ++i) {
      (*xx->stats_out)[2 * rc[i].orig] += (double)st[3 * i];
      (*xx->stats_out)[2 * rc[i].orig + 1] += (double)st[3 * i + 2];
    }
  }
  return PROTEA_OK;
}

}  // namespace

extern "C" {

protea_status protea_run_round(protea_ctx* ctx, const protea_round_opts* opts, const protea_client* clients, size_t n,
                               const protea_assignment* plan, const float* global_in, float* global_out,
                               size_t n_params, protea_profile* measured, protea_round_stats* stats) {
  if (!ctx) return PROTEA_ERR_INVALID;
  int64_t Ptot = 0;
  for (auto& g : ctx->groups) Ptot += g.m.P;
  const int e = ctx->precision == PROTEA_PREC_FP32 ? 4 : 2;
  std::vector<RunClient> all;
  std::vector<int64_t> Ngroup(ctx->groups.size(), 0);
  // ---- validate clients and plan (every check of this rank; with a communicator the verdict is agreed
  // on by all ranks below before any of them starts device work, so one rank's failure cannot leave
  // the others waiting in a collective)
  auto validate = [&]() -> protea_status {
    if (!opts || !clients || !plan || !global_in || !global_out || n == 0)
      return fail(ctx, PROTEA_ERR_INVALID, "run_round: null argument or n == 0");
    if ((int64_t)n_params != Ptot)
      return fail(ctx, PROTEA_ERR_DIM, "run_round: n_params " + std::to_string(n_params) + " != registered total " +
                                           std::to_string(Ptot));
    std::map<int64_t, const protea_assignment*> pa;
    for (size_t i = 0; i < n; ++i)
      if (!pa.emplace(plan[i].client_id, &plan[i]).second)
        return fail(ctx, PROTEA_ERR_PLAN, "run_round: plan lists client " + std::to_string(plan[i].client_id) + " twice");
    std::map<int64_t, int> seen;
    for (size_t i = 0; i < n; ++i) {
      const protea_client& c = clients[i];
      const std::string who = "run_round: client " + std::to_string(c.client_id);
      if (!seen.emplace(c.client_id, 1).second) return fail(ctx, PROTEA_ERR_INVALID, who + " listed twice");
      if (c.model_id < 0 || c.model_id >= (int)ctx->groups.size())
        return fail(ctx, PROTEA_ERR_INVALID, who + ": unknown model_id");
      if (c.batch <= 0 || c.batch > kMaxBatch || c.epochs <= 0)
        return fail(ctx, PROTEA_ERR_INVALID, who + ": batch must be in [1, " + std::to_string(kMaxBatch) +
                                                 "] and epochs > 0");
      auto sh = ctx->shards.find(c.client_id);
      if (sh == ctx->shards.end()) return fail(ctx, PROTEA_ERR_INVALID, who + ": no registered shard");
      if (sh->second.ymin < 0 || sh->second.ymax >= ctx->groups[c.model_id].m.classes)
        return fail(ctx, PROTEA_ERR_INVALID, who + ": label outside [0, " +
                                                 std::to_string(ctx->groups[c.model_id].m.classes) + ")");
      auto it = pa.find(c.client_id);
      if (it == pa.end()) return fail(ctx, PROTEA_ERR_PLAN, who + " missing from the plan");
      const protea_assignment& a = *it->second;
      RunClient r;
      r.id = c.client_id;
      r.group = c.model_id;
      r.n = sh->second.n;
      r.B = c.batch;
      r.E = c.epochs;
      r.nb = (int)ceil_div((uint64_t)r.n, (uint64_t)r.B);
      r.S = (uint64_t)r.E * r.nb;
      r.admit = a.admit;
      r.release = a.release;
      r.offset = a.offset;
      r.slot = a.slot;
      if (a.gpu < 0 || a.gpu >= ctx->world) return fail(ctx, PROTEA_ERR_PLAN, who + ": gpu out of range");
      if (a.release != a.admit + r.S)
        return fail(ctx, PROTEA_ERR_PLAN, who + ": release - admit != S_k = " + std::to_string(r.S));
      const uint64_t need = client_hwm(ctx->groups[c.model_id].m, r.B, r.n, r.E, e);
      if (a.slot < need)
        return fail(ctx, PROTEA_ERR_PLAN, who + ": slot " + std::to_string(a.slot) + " < HWM " + std::to_string(need));
      if (a.gpu == ctx->rank && (a.offset % kAlign != 0 || a.offset + a.slot > ctx->arena_bytes))
        return fail(ctx, PROTEA_ERR_OOM, who + ": slot [" + std::to_string(a.offset) + ", +" + std::to_string(a.slot) +
                                             ") outside the arena of " + std::to_string(ctx->arena_bytes) + " B");
      Ngroup[c.model_id] += r.n;
      if (a.gpu == ctx->rank) all.push_back(r);
    }
    if (pa.size() != n) return fail(ctx, PROTEA_ERR_PLAN, "run_round: plan and client list differ");
    if (opts->n_trace && (!opts->trace_ids || !opts->trace_bufs))
      return fail(ctx, PROTEA_ERR_INVALID, "run_round: n_trace > 0 with null trace_ids / trace_bufs");
    for (uint32_t i = 0; i < opts->n_trace; ++i) {
      auto it = std::find_if(all.begin(), all.end(), [&](const RunClient& c) { return c.id == opts->trace_ids[i]; });
      if (it == all.end() || !opts->trace_bufs[i] || !is_device_ptr(opts->trace_bufs[i]))
        return fail(ctx, PROTEA_ERR_INVALID, "run_round: traced client " + std::to_string(opts->trace_ids[i]) +
                                                 " is not one of this rank's clients or has no device buffer");
    }
    // live slots pairwise disjoint on this GPU
    std::vector<RunClient*> byoff;
    for (auto& c : all) byoff.push_back(&c);
    std::sort(byoff.begin(), byoff.end(), [](RunClient* a, RunClient* b) { return a->offset < b->offset; });
    for (size_t i = 0; i < byoff.size(); ++i)
      for (size_t j = i + 1; j < byoff.size(); ++j) {
        RunClient* a = byoff[i];
        RunClient* b = byoff[j];
        const uint64_t aend = a->offset + client_hwm(ctx->groups[a->group].m, a->B, a->n, a->E, e);
        if (b->offset >= aend) break;
        if (a->admit < b->release && b->admit < a->release)
          return fail(ctx, PROTEA_ERR_PLAN, "run_round: clients " + std::to_string(a->id) + " and " +
                                                std::to_string(b->id) + " overlap in the arena while both live");
      }
    return PROTEA_OK;
  };
  NvtxRange nv_round("protea_run_round");
  protea_status vst;
  {
    NvtxRange nv("protea: validate");
    vst = validate();
  }
  if (ctx->comm) {
    // plan agreement + validation verdict: NCCL max over ranks of (h, ~h, failed) equals
    // (h, ~h, 0) iff every rank validated and all ranks hold the same client list and plan
    const uint64_t h = vst == PROTEA_OK ? protea_plan_hash(clients, n, plan) : 0;
    const uint64_t flag = vst == PROTEA_OK ? 0 : 1;
    const uint64_t hv0[3] = {h, ~h, flag};
    uint64_t hv[3];
    std::memcpy(hv, hv0, sizeof(hv));
    CK(cudaSetDevice(ctx->device));
    CK(ctx->flag.reserve(4));
    CK(cudaMemcpyAsync(ctx->flag.p, hv, 24, cudaMemcpyHostToDevice, ctx->stream));
    ncclResult_t r = ncclAllReduce(ctx->flag.p, ctx->flag.p, 3, ncclUint64, ncclMax, ctx->comm, ctx->stream);
    if (r != ncclSuccess) return fail(ctx, PROTEA_ERR_NCCL, std::string("run_round: plan hash allreduce: ") + ncclGetErrorString(r));
    CK(cudaMemcpyAsync(hv, ctx->flag.p, 24, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (vst != PROTEA_OK) return vst;
    if (hv[2]) return fail(ctx, PROTEA_ERR_PLAN, "run_round: another rank rejected the round (validation)");
    if (hv[0] != hv0[0] || hv[1] != hv0[1])
      return fail(ctx, PROTEA_ERR_PLAN, "run_round: ranks disagree on the plan / client list (plan hash)");
  } else if (vst != PROTEA_OK) {
    return vst;
  }
  std::sort(all.begin(), all.end(), [](const RunClient& a, const RunClient& b) { return a.id < b.id; });
  CK(cudaSetDevice(ctx->device));
  // ---- global weights in
  const bool in_dev = is_device_ptr(global_in), out_dev = is_device_ptr(global_out);
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  const float* wg = global_in;
  if (!in_dev) {
    CK(ctx->gin.reserve(Ptot));
    CK(cudaMemcpyAsync(ctx->gin.p, global_in, Ptot * 4, cudaMemcpyHostToDevice, ctx->stream));
    wg = ctx->gin.p;
  } else if (global_in == global_out) {
    // finalize writes out while admissions of later iterations are done; keep a private copy
    CK(ctx->gin.reserve(Ptot));
    CK(cudaMemcpyAsync(ctx->gin.p, global_in, Ptot * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    wg = ctx->gin.p;
  }
  const size_t NG = ctx->groups.size();  // one fp64 loss-sum slot per group after the accumulators
  CK(ctx->acc.reserve(Ptot + NG));
  CK(cudaMemsetAsync(ctx->acc.p, 0, (Ptot + NG) * 8, ctx->stream));
  reset_ops(ctx, opts->time_ops);
  ctx->serialize = opts->serialize != 0;
  const uint64_t l0 = ctx->launches;
  uint64_t iters = 0;
  double* loss_dev = ctx->acc.p + Ptot;  // per-group fp64 sums of step losses after the accumulators
  ExecExtras xx;
  xx.observe = opts->observe_hwm != 0;
  for (uint32_t i = 0; i < opts->n_trace; ++i) xx.trace[opts->trace_ids[i]] = (uint8_t*)opts->trace_bufs[i];
  protea_status st;
  {
    NvtxRange nv("protea: execute (A2 local SGD, A3 profiles, A5 FedAvg accumulation)");
    st = execute(ctx, all, wg, ctx->acc.p, opts->lr, opts->seed, opts->round, opts->shuffle, &iters, loss_dev, &xx);
  }
  NvtxRange nv_x("protea: exchange + finalise (K7)");
  if (ctx->comm && !opts->partial_only) {
    // every rank reaches the exchange; one that failed inside execute() says so first (NCCL max of a flag)
    const uint64_t f0 = st == PROTEA_OK ? 0 : 1;
    uint64_t f = f0;
    CK(ctx->flag.reserve(4));
    CK(cudaMemcpyAsync(ctx->flag.p, &f, 8, cudaMemcpyHostToDevice, ctx->stream));
    ncclResult_t r = ncclAllReduce(ctx->flag.p, ctx->flag.p, 1, ncclUint64, ncclMax, ctx->comm, ctx->stream);
    if (r != ncclSuccess) return fail(ctx, PROTEA_ERR_NCCL, std::string("run_round: error-flag allreduce: ") + ncclGetErrorString(r));
    CK(cudaMemcpyAsync(&f, ctx->flag.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (st != PROTEA_OK) return st;
    if (f) return fail(ctx, PROTEA_ERR_CUDA, "run_round: another rank failed during the round");
  }
  if (st != PROTEA_OK) return st;
  ctx->last_Ngroup = Ngroup;
  ctx->have_partial = opts->partial_only != 0;
  if (opts->partial_only) {
    CK(cudaEventRecord(ctx->ev1, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (stats) {
      float pms = 0.f;
      CK(cudaEventElapsedTime(&pms, ctx->ev0, ctx->ev1));
      std::memset(stats, 0, sizeof(*stats));
      stats->round_ns = (uint64_t)(pms * 1e6);
      stats->iterations = iters;
      stats->kernel_launches = ctx->launches - l0;
      for (auto& c : all) stats->client_steps += c.S;
    }
    return PROTEA_OK;
  }
  if (ctx->world > 1 && !ctx->comm)
    return fail(ctx, PROTEA_ERR_INVALID, "run_round: world > 1 without an NCCL communicator needs partial_only = 1");
  // K7: the ranks' fp64 partials (and per-group loss sums) are all-gathered and every rank
  // sums them in RANK ORDER inside the finalise kernel, so the result is bitwise defined for a given
  // world size (an ncclAllReduce sum would leave the order to NCCL's algorithm choice)
  const int64_t stride = Ptot + (int64_t)NG;
  const double* parts = ctx->acc.p;
  int nparts = 1;
  if (ctx->comm) {
    CK(ctx->gath.reserve((size_t)stride * ctx->world));
    ncclResult_t r = ncclAllGather(ctx->acc.p, ctx->gath.p, stride, ncclDouble, ctx->comm, ctx->stream);
    if (r != ncclSuccess) return fail(ctx, PROTEA_ERR_NCCL, std::string("run_round: ncclAllGather: ") + ncclGetErrorString(r));
    parts = ctx->gath.p;
    nparts = ctx->world;
  }
  float* out = global_out;
  if (!out_dev) {
    CK(ctx->gout.reserve(Ptot));
    out = ctx->gout.p;
  }
  for (size_t g = 0; g < ctx->groups.size(); ++g) {
    const Group& gr = ctx->groups[g];
    if (Ngroup[g] > 0) {
      ctx->op_bytes[PROTEA_OPC_FEDAVG] += (8 * (uint64_t)nparts + 8) * (uint64_t)gr.m.P;
      const int ev = op_begin(ctx, PROTEA_OPC_FEDAVG);
      k_finalize_ordered<<<grid_for(gr.m.P, 256), 256, 0, ctx->stream>>>(
          wg + gr.offset, parts + gr.offset, stride, nparts, (double)Ngroup[g], out + gr.offset, gr.m.P);
      op_end(ctx, ev);
    } else if (out + gr.offset != wg + gr.offset) {
      CK(cudaMemcpyAsync(out + gr.offset, wg + gr.offset, gr.m.P * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    }
  }
  if (!out_dev) CK(cudaMemcpyAsync(global_out, out, Ptot * 4, cudaMemcpyDeviceToHost, ctx->stream));
  std::vector<double> loss_g((size_t)nparts * NG, 0.0);
  CK(cudaMemcpy2DAsync(loss_g.data(), NG * 8, parts + Ptot, (size_t)stride * 8, NG * 8, nparts,
                       cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  double loss_sum = 0.0;
  for (double v : loss_g) loss_sum += v;  // rank order, group order
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->round_ns = (uint64_t)(ms * 1e6);
    stats->iterations = iters;
    stats->kernel_launches = ctx->launches - l0;
    stats->loss_sum = loss_sum;
    for (int i = 0; i < PROTEA_N_OPC; ++i) {
      stats->op_launches[i] = ctx->op_launches[i];
      stats->op_flops[i] = ctx->op_flops[i];
      stats->op_bytes[i] = ctx->op_bytes[i];
    }
    for (size_t k = 0; k < ctx->ev_op.size(); ++k) {
      float ems = 0.f;
      CK(cudaEventElapsedTime(&ems, ctx->evpool[2 * k], ctx->evpool[2 * k + 1]));
      stats->op_ns[ctx->ev_op[k]] += (uint64_t)((double)ems * 1e6);
      stats->op_timed_launches[ctx->ev_op[k]]++;
      stats->op_timed_flops[ctx->ev_op[k]] += ctx->ev_work[k].first;
      stats->op_timed_bytes[ctx->ev_op[k]] += ctx->ev_work[k].second;
    }
    for (auto& c : all) {
      stats->client_steps += c.S;
      stats->flops += (uint64_t)c.E * c.n * flops_per_sample(ctx->groups[c.group].m);
    }
  }
  std::vector<uint64_t> smns(all.size(), 0);
  if (!all.empty()) CK(cudaMemcpy(smns.data(), ctx->smns.p, all.size() * 8, cudaMemcpyDeviceToHost));
  std::map<int64_t, uint64_t> sm_of, hwm_of;
  for (size_t i = 0; i < all.size(); ++i) sm_of[all[i].id] = smns[i];
  if (xx.observe && !all.empty()) {
    std::vector<uint64_t> h(all.size(), 0);
    CK(cudaMemcpy(h.data(), ctx->hwm.p, all.size() * 8, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < all.size(); ++i) hwm_of[all[i].id] = align256(h[i]);
  }
  if (measured) {
    size_t k = 0;
    for (size_t i = 0; i < n; ++i) {
      const protea_client& c = clients[i];
      const int64_t nn = ctx->shards[c.client_id].n;
      protea_profile& p = measured[k++];
      std::memset(&p, 0, sizeof(p));
      p.client_id = c.client_id;
      p.peak_bytes = client_hwm(ctx->groups[c.model_id].m, c.batch, nn, c.epochs, e);
      auto ho = hwm_of.find(c.client_id);  // observe_hwm: this rank's clients report the observed mark
      if (ho != hwm_of.end()) p.peak_bytes = ho->second;
      p.steps = (uint64_t)c.epochs * ceil_div((uint64_t)nn, (uint64_t)c.batch);
      p.flops = (uint64_t)c.epochs * nn * flops_per_sample(ctx->groups[c.model_id].m);
      p.uses_gpu = 1;
      auto it = sm_of.find(c.client_id);  // clients of other ranks keep 0
      if (it != sm_of.end()) {
        p.sm_ns = it->second;
        p.train_ns = it->second / (uint64_t)g_num_sms;  // SM-time share expressed as whole-GPU time
        p.step_ns = p.steps ? p.train_ns / p.steps : 0;
      }
    }
  }
  return PROTEA_OK;
}

protea_status protea_profile_clients(protea_ctx* ctx, const protea_client* clients, size_t n, protea_profile* out) {
  if (!ctx) return PROTEA_ERR_INVALID;
  if (!clients || !out || n == 0) return fail(ctx, PROTEA_ERR_INVALID, "profile_clients: null argument or n == 0");
  const int e = ctx->precision == PROTEA_PREC_FP32 ? 4 : 2;
  std::map<std::pair<int, int>, uint64_t> class_ns;  // (model, batch) -> probe step ns
  for (size_t i = 0; i < n; ++i) {
    const protea_client& c = clients[i];
    const std::string who = "profile_clients: client " + std::to_string(c.client_id);
    if (c.model_id < 0 || c.model_id >= (int)ctx->groups.size())
      return fail(ctx, PROTEA_ERR_INVALID, who + ": unknown model_id");
    if (c.batch <= 0 || c.batch > kMaxBatch || c.epochs <= 0)
      return fail(ctx, PROTEA_ERR_INVALID, who + ": batch must be in [1, " + std::to_string(kMaxBatch) + "] and epochs > 0");
    auto sh = ctx->shards.find(c.client_id);
    if (sh == ctx->shards.end()) return fail(ctx, PROTEA_ERR_INVALID, who + ": no registered shard");
    if (sh->second.ymin < 0 || sh->second.ymax >= ctx->groups[c.model_id].m.classes)
      return fail(ctx, PROTEA_ERR_INVALID, who + ": label outside [0, " +
                                               std::to_string(ctx->groups[c.model_id].m.classes) + ")");
  }
  CK(cudaSetDevice(ctx->device));
  for (size_t i = 0; i < n; ++i) {
    const protea_client& c = clients[i];
    auto key = std::make_pair((int)c.model_id, (int)c.batch);
    if (class_ns.count(key)) continue;
    // probe: this client alone at arena offset 0, timed (CUDA events) as a one-step and a two-step run;
    // step_ns is the DIFFERENCE of the medians, i.e. the marginal cost of a local step without the
    // admission, permutation and host-table upload every run pays once
    const Group& gr = ctx->groups[c.model_id];
    RunClient r;
    r.id = c.client_id;
    r.group = c.model_id;
    r.n = std::max<int64_t>(ctx->shards[c.client_id].n, 1);
    r.B = c.batch;
    r.nb = (int)ceil_div((uint64_t)r.n, (uint64_t)r.B);
    r.E = r.nb >= 2 ? 1 : 2;  // the second step exists within this client's own schedule
    r.admit = 0;
    r.offset = 0;
    const uint64_t need = client_hwm(gr.m, r.B, r.n, r.E, e);
    if (need > ctx->arena_bytes)
      return fail(ctx, PROTEA_ERR_OOM, "profile_clients: probe slot of " + std::to_string(need) +
                                           " B exceeds the arena");
    CK(ctx->gin.reserve(gr.m.P));
    CK(cudaMemsetAsync(ctx->gin.p, 0, gr.m.P * 4, ctx->stream));
    reset_ops(ctx, 0);
    float med[2];
    for (int steps = 1; steps <= 2; ++steps) {
      r.S = steps;
      r.release = steps;
      std::vector<float> times;
      for (int rep = 0; rep < 7; ++rep) {
        std::vector<RunClient> one{r};
        // gin holds zero weights at offset 0; shift so that wg + group offset == gin
        const float* wg = ctx->gin.p - gr.offset;
        CK(cudaEventRecord(ctx->ev0, ctx->stream));
        protea_status st = execute(ctx, one, wg, nullptr, 0.0f, 0, 0, 0, nullptr, nullptr);
        if (st != PROTEA_OK) return st;
        CK(cudaEventRecord(ctx->ev1, ctx->stream));
        CK(cudaEventSynchronize(ctx->ev1));
        float ms;
        CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        if (rep >= 2) times.push_back(ms);
      }
      std::sort(times.begin(), times.end());
      med[steps - 1] = times[times.size() / 2];
    }
    // a difference of medians can be <= 0 under noise for very cheap steps: floor at 1 us
    class_ns[key] = (uint64_t)std::max(1e3, (double)(med[1] - med[0]) * 1e6);
  }
  // ---- observed high-water marks: every client runs ONE local step (admission with its E epoch
  // permutations, one batch of min(B, n_k) rows) in a poisoned slot of the layout's size followed by a
  // poisoned guard; clients are packed back to back, as many per lock-step probe as the arena holds
  std::vector<uint64_t> observed(n, 0);
  {
    constexpr uint64_t kGuard = 4096;
    std::vector<uint64_t> need(n);
    for (size_t i = 0; i < n; ++i)
      need[i] = client_hwm(ctx->groups[clients[i].model_id].m, clients[i].batch, ctx->shards[clients[i].client_id].n,
                           clients[i].epochs, e);
    int64_t Pmax = 0;
    for (auto& g : ctx->groups) Pmax = std::max<int64_t>(Pmax, g.m.P);
    size_t i0 = 0;
    while (i0 < n) {
      std::vector<RunClient> batch;
      std::vector<size_t> idx;
      std::vector<uint64_t> reg;
      std::map<int64_t, int> ids_in;
      uint64_t off = 0;
      size_t i1 = i0;
      while (i1 < n && off + need[i1] + kGuard <= ctx->arena_bytes) {
        const protea_client& c = clients[i1];
        if (ids_in.count(c.client_id)) break;  // one record per client id per probe
        ids_in[c.client_id] = 1;
        RunClient r;
        r.id = c.client_id;
        r.group = c.model_id;
        r.n = ctx->shards[c.client_id].n;
        r.B = c.batch;
        r.E = c.epochs;
        r.nb = (int)ceil_div((uint64_t)r.n, (uint64_t)r.B);
        r.S = 1;
        r.admit = 0;
        r.release = 1;
        r.offset = off;
        r.slot = need[i1];
        const uint64_t k2 = 2 * batch.size();  // (offset, bytes, output index): the slot, then its guard
        reg.insert(reg.end(), {off, need[i1], k2, off + need[i1], kGuard, k2 + 1});
        off += need[i1] + kGuard;
        batch.push_back(r);
        idx.push_back(i1);
        ++i1;
      }
      if (batch.empty())
        return fail(ctx, PROTEA_ERR_OOM, "profile_clients: client " + std::to_string(clients[i0].client_id) +
                                             ": slot of " + std::to_string(need[i0]) + " B + guard exceeds the arena");
      CK(cudaMemsetAsync(ctx->arena, PROTEA_POISON, off, ctx->stream));
      CK(ctx->gin.reserve(Pmax));
      CK(cudaMemsetAsync(ctx->gin.p, 0, Pmax * 4, ctx->stream));
      // every group reads its global weights at gin + group offset - offset: zero weights for all
      std::vector<RunClient> order(batch);
      std::sort(order.begin(), order.end(), [](const RunClient& a, const RunClient& b) { return a.id < b.id; });
      std::vector<std::vector<RunClient>> by_group(ctx->groups.size());
      for (auto& r : order) by_group[r.group].push_back(r);
      for (size_t g = 0; g < ctx->groups.size(); ++g) {
        if (by_group[g].empty()) continue;
        const float* wg = ctx->gin.p - ctx->groups[g].offset;
        reset_ops(ctx, 0);
        protea_status st = execute(ctx, by_group[g], wg, nullptr, 0.0f, 0, 0, 1, nullptr, nullptr);
        if (st != PROTEA_OK) return st;
      }
      const size_t nreg = reg.size() / 3;
      CK(ctx->regions.reserve(reg.size()));
      CK(ctx->hwm.reserve(nreg));
      CK(cudaMemcpyAsync(ctx->regions.p, reg.data(), reg.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemsetAsync(ctx->hwm.p, 0, nreg * 8, ctx->stream));
      uint64_t max_reg = 0;
      for (size_t k = 1; k < reg.size(); k += 3) max_reg = std::max(max_reg, reg[k]);
      k_scan_poison<<<dim3(grid_for((int64_t)(max_reg / 16), 256, 2 * g_num_sms), (unsigned)nreg), 256, 0,
                      ctx->stream>>>(ctx->arena, ctx->regions.p, nullptr, ctx->hwm.p);
      CK(cudaGetLastError());
      std::vector<uint64_t> h(nreg);
      CK(cudaMemcpyAsync(h.data(), ctx->hwm.p, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      for (size_t k = 0; k < batch.size(); ++k) {
        if (h[2 * k + 1])
          return fail(ctx, PROTEA_ERR_OOM, "profile_clients: client " + std::to_string(batch[k].id) +
                                               " wrote " + std::to_string(h[2 * k + 1]) +
                                               " B past its slot (guard canary touched)");
        observed[idx[k]] = align256(h[2 * k]);
      }
      i0 = i1;
    }
  }
  for (size_t i = 0; i < n; ++i) {
    const protea_client& c = clients[i];
    const int64_t nn = ctx->shards[c.client_id].n;
    protea_profile& p = out[i];
    std::memset(&p, 0, sizeof(p));
    p.client_id = c.client_id;
    p.peak_bytes = observed[i];
    p.steps = (uint64_t)c.epochs * ceil_div((uint64_t)nn, (uint64_t)c.batch);
    p.flops = (uint64_t)c.epochs * nn * flops_per_sample(ctx->groups[c.model_id].m);
    p.step_ns = class_ns[std::make_pair((int)c.model_id, (int)c.batch)];
    p.train_ns = p.step_ns * p.steps;
    p.uses_gpu = 1;
  }
  return PROTEA_OK;
}

protea_status protea_round_partial(protea_ctx* ctx, double* dst, size_t n_params) {
  if (!ctx) return PROTEA_ERR_INVALID;
  int64_t Ptot = 0;
  for (auto& g : ctx->groups) Ptot += g.m.P;
  if (!dst || !ctx->have_partial) return fail(ctx, PROTEA_ERR_INVALID, "round_partial: no partial round recorded");
  if ((int64_t)n_params != Ptot) return fail(ctx, PROTEA_ERR_DIM, "round_partial: n_params mismatch");
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpyAsync(dst, ctx->acc.p, Ptot * 8, cudaMemcpyDefault, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return PROTEA_OK;
}

protea_status protea_round_finalize_ordered(protea_ctx* ctx, const double* partials, int32_t nparts,
                                            const float* global_in, float* global_out, size_t n_params) {
  if (!ctx) return PROTEA_ERR_INVALID;
  if (!partials || !global_in || !global_out || nparts < 1 || ctx->last_Ngroup.size() != ctx->groups.size())
    return fail(ctx, PROTEA_ERR_INVALID, "round_finalize: null argument, nparts < 1 or no round recorded");
  int64_t Ptot = 0;
  for (auto& g : ctx->groups) Ptot += g.m.P;
  if ((int64_t)n_params != Ptot) return fail(ctx, PROTEA_ERR_DIM, "round_finalize: n_params mismatch");
  CK(cudaSetDevice(ctx->device));
  CK(ctx->gin.reserve(Ptot));
  CK(ctx->gout.reserve(Ptot));
  CK(ctx->gath.reserve((size_t)Ptot * nparts));
  CK(cudaMemcpyAsync(ctx->gin.p, global_in, Ptot * 4, cudaMemcpyDefault, ctx->stream));
  CK(cudaMemcpyAsync(ctx->gath.p, partials, (size_t)Ptot * nparts * 8, cudaMemcpyDefault, ctx->stream));
  for (size_t g = 0; g < ctx->groups.size(); ++g) {
    const Group& gr = ctx->groups[g];
    if (ctx->last_Ngroup[g] > 0)
      k_finalize_ordered<<<grid_for(gr.m.P, 256), 256, 0, ctx->stream>>>(
          ctx->gin.p + gr.offset, ctx->gath.p + gr.offset, Ptot, nparts, (double)ctx->last_Ngroup[g],
          ctx->gout.p + gr.offset, gr.m.P);
    else
      CK(cudaMemcpyAsync(ctx->gout.p + gr.offset, ctx->gin.p + gr.offset, gr.m.P * 4, cudaMemcpyDeviceToDevice,
                         ctx->stream));
  }
  CK(cudaMemcpyAsync(global_out, ctx->gout.p, Ptot * 4, cudaMemcpyDefault, ctx->stream));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->have_partial = false;
  return PROTEA_OK;
}

protea_status protea_round_finalize(protea_ctx* ctx, const double* acc_sum, const float* global_in, float* global_out,
                                    size_t n_params) {
  return protea_round_finalize_ordered(ctx, acc_sum, 1, global_in, global_out, n_params);
}

protea_status protea_evaluate(protea_ctx* ctx, int32_t model_id, const float* weights, const uint8_t* x,
                              const int32_t* y, int64_t n, protea_eval_result* out) {
  if (!ctx) return PROTEA_ERR_INVALID;
  if (!weights || !x || !y || !out) return fail(ctx, PROTEA_ERR_INVALID, "evaluate: null pointer");
  if (n <= 0) return fail(ctx, PROTEA_ERR_INVALID, "evaluate: n must be > 0");
  if (model_id < 0 || model_id >= (int)ctx->groups.size()) return fail(ctx, PROTEA_ERR_INVALID, "evaluate: unknown model_id");
  const ModelDims& m = ctx->groups[model_id].m;
  if (m.arch != PROTEA_MODEL_CNN && m.arch != PROTEA_MODEL_MLP)
    return fail(ctx, PROTEA_ERR_INVALID, "evaluate: MLP and CNN models only");
  for (int64_t i = 0; i < n; ++i)
    if (y[i] < 0 || y[i] >= m.classes)
      return fail(ctx, PROTEA_ERR_INVALID, "evaluate: label of sample " + std::to_string(i) + " outside [0, classes)");
  CK(cudaSetDevice(ctx->device));
  constexpr int RB = 64;  // samples per group (one task of the grouped forward launches)
  const int T = (int)cdiv(n, RB);
  const int64_t D = m.in_dim(), P = m.P;
  // per-group activation buffers (fp32 verify-mode layout, slot_layout sizes at batch RB)
  const SlotLayout sl = slot_layout(m, RB, RB, 1, 4);
  std::vector<int> used;
  for (int b : {B_A1, B_I1, B_A2, B_I2, B_H, B_H1})
    if (sl.used[b]) used.push_back(b);
  uint64_t per = 0;
  for (int b : used) per += align256(sl.size[b]);
  const uint64_t off_w = 0, off_x = align256(4 * (uint64_t)P), off_y = off_x + align256((uint64_t)n * D),
                 off_p = off_y + align256(4 * (uint64_t)n), off_a = off_p + align256(4 * (uint64_t)n);
  CK(ctx->ev_ws.reserve(off_a + per * T));
  uint8_t* ws = ctx->ev_ws.p;
  cudaStream_t st = ctx->stream;
  CK(cudaMemcpyAsync(ws + off_w, weights, 4 * (size_t)P, is_device_ptr(weights) ? cudaMemcpyDeviceToDevice
                                                                                  : cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ws + off_x, x, (size_t)n * D, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ws + off_y, y, 4 * (size_t)n, cudaMemcpyHostToDevice, st));
  std::vector<int32_t> ident(n);
  for (int64_t i = 0; i < n; ++i) ident[i] = (int32_t)i;
  CK(cudaMemcpyAsync(ws + off_p, ident.data(), 4 * (size_t)n, cudaMemcpyHostToDevice, st));
  std::vector<ClientRec> recs(T);
  for (int t = 0; t < T; ++t) {
    ClientRec& r = recs[t];
    std::memset(&r, 0, sizeof(r));
    r.params = (float*)(ws + off_w);
    r.perm = (int32_t*)(ws + off_p);
    r.x = ws + off_x;
    r.y = (const int32_t*)(ws + off_y);
    r.n = (int32_t)n;
    r.B = RB;
    r.E = 1;
    r.nb = T;
    r.P = P;
    r.c1 = m.c1;
    uint64_t o = off_a + per * t;
    for (int b : used) {
      r.buf[b] = ws + o;
      o += align256(sl.size[b]);
    }
  }
  // schedule table: T tasks (rec t, step 0, rows, base 64 t) and the forward ops' prefix arrays
  const std::vector<int> ops = m.arch == PROTEA_MODEL_CNN ? std::vector<int>{OP_C1F, OP_C2F, OP_F1F}
                                                          : std::vector<int>{OP_MF};
  std::vector<int32_t> tab;
  Launch L;
  std::memset(&L, 0, sizeof(L));
  L.ntask = T;
  L.task_off = 0;
  std::vector<int> rows(T);
  for (int t = 0; t < T; ++t) {
    rows[t] = (int)std::min<int64_t>(RB, n - (int64_t)t * RB);
    tab.insert(tab.end(), {t, 0, rows[t], t * RB});
  }
  for (int op : ops) {
    L.prefix_off[op] = (int64_t)tab.size();
    int acc_t = 0;
    for (int t = 0; t < T; ++t) {
      tab.push_back(acc_t);
      acc_t += tiles(m, op, rows[t], false);
    }
    tab.push_back(acc_t);
    L.grid[op] = acc_t;
  }
  CK(ctx->ev_recs.reserve(T));
  CK(ctx->ev_tab.reserve(tab.size()));
  CK(ctx->ev_loss.reserve(T));
  CK(ctx->ev_ok.reserve(T));
  CK(cudaMemcpyAsync(ctx->ev_recs.p, recs.data(), T * sizeof(ClientRec), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->ev_tab.p, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice, st));
  const ClientRec* drecs = ctx->ev_recs.p;
  const int32_t* dtab = ctx->ev_tab.p;
  const Task* tasks = reinterpret_cast<const Task*>(dtab);
  ctx->cur = st;
  const uint32_t keep_time = ctx->time_ops;
  ctx->time_ops = 0;
  if (m.arch == PROTEA_MODEL_CNN) {
    const CnnDims d = cnn_dims(m);
    launch_gemm<Conv1Fwd<float, C1F_BM, C1F_BN>, C1F_BM, C1F_BN>(ctx, {drecs, d}, L, OP_C1F, dtab);
    launch_gemm<Conv2Fwd<float, C2F_BM, C2F_BN>, C2F_BM, C2F_BN>(ctx, {drecs, d}, L, OP_C2F, dtab);
    launch_gemm<Fc1Fwd<float, F1F_BM, F1F_BN>, F1F_BM, F1F_BN>(ctx, {drecs, d}, L, OP_F1F, dtab);
    k_eval_head<float><<<T, 256, 0, st>>>(drecs, tasks, B_H, m.f, m.classes, d.w4, d.b4, ctx->ev_loss.p,
                                          ctx->ev_ok.p);
  } else {
    const MlpDims d = mlp_dims(m);
    launch_gemm<MlpFc1Fwd<float, MF_BM, MF_BN>, MF_BM, MF_BN>(ctx, {drecs, d}, L, OP_MF, dtab);
    k_eval_head<float><<<T, 256, 0, st>>>(drecs, tasks, B_H1, 64, m.classes, d.w2, d.b2, ctx->ev_loss.p,
                                          ctx->ev_ok.p);
  }
  ctx->time_ops = keep_time;
  CK(cudaGetLastError());
  std::vector<double> lo(T);
  std::vector<uint32_t> ok(T);
  CK(cudaMemcpyAsync(lo.data(), ctx->ev_loss.p, T * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(ok.data(), ctx->ev_ok.p, T * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  out->loss_sum = 0.0;
  out->correct = 0;
  for (int t = 0; t < T; ++t) {  // fixed group order: deterministic
    out->loss_sum += lo[t];
    out->correct += ok[t];
  }
  out->n = (uint64_t)n;
  return PROTEA_OK;
}

protea_status protea_evaluate_round(protea_ctx* ctx, const protea_client* clients, size_t n, const float* global,
                                    size_t n_params, protea_eval_result* per_client, protea_eval_result* total) {
  if (!ctx) return PROTEA_ERR_INVALID;
  if (!clients || !global || !per_client || n == 0)
    return fail(ctx, PROTEA_ERR_INVALID, "evaluate_round: null argument or n == 0");
  int64_t Ptot = 0;
  for (auto& g : ctx->groups) Ptot += g.m.P;
  if ((int64_t)n_params != Ptot) return fail(ctx, PROTEA_ERR_DIM, "evaluate_round: n_params mismatch");
  const int e = ctx->precision == PROTEA_PREC_FP32 ? 4 : 2;
  std::map<int64_t, int> seen;
  for (size_t i = 0; i < n; ++i) {
    const protea_client& c = clients[i];
    const std::string who = "evaluate_round: client " + std::to_string(c.client_id);
    if (!seen.emplace(c.client_id, 1).second) return fail(ctx, PROTEA_ERR_INVALID, who + " listed twice");
    if (c.model_id < 0 || c.model_id >= (int)ctx->groups.size())
      return fail(ctx, PROTEA_ERR_INVALID, who + ": unknown model_id");
    auto sh = ctx->val_shards.find(c.client_id);
    if (sh == ctx->val_shards.end()) return fail(ctx, PROTEA_ERR_INVALID, who + ": no registered validation split");
    if (sh->second.ymin < 0 || sh->second.ymax >= ctx->groups[c.model_id].m.classes)
      return fail(ctx, PROTEA_ERR_INVALID, who + ": label outside [0, classes)");
  }
  CK(cudaSetDevice(ctx->device));
  const float* wg = global;
  if (!is_device_ptr(global)) {
    CK(ctx->gin.reserve(Ptot));
    CK(cudaMemcpyAsync(ctx->gin.p, global, Ptot * 4, cudaMemcpyHostToDevice, ctx->stream));
    wg = ctx->gin.p;
  }
  // every client evaluates its group's global weights on its whole validation split: one lock-step
  // "step" per batch of up to kMaxBatch rows (micro-clients above kMicroRows), slots packed back to back
  // in the arena, as many clients per pass as it holds
  size_t i0 = 0;
  while (i0 < n) {
    std::vector<RunClient> batch;
    std::vector<size_t> idx;
    uint64_t off = 0;
    size_t i1 = i0;
    while (i1 < n) {
      const protea_client& c = clients[i1];
      RunClient r;
      r.id = c.client_id;
      r.group = c.model_id;
      r.n = ctx->val_shards[c.client_id].n;
      r.B = (int)std::min<int64_t>(r.n, kMaxBatch);
      r.E = 1;
      r.nb = (int)ceil_div((uint64_t)r.n, (uint64_t)r.B);
      r.S = r.nb;
      r.admit = 0;
      r.release = r.S;
      const uint64_t need = client_hwm(ctx->groups[c.model_id].m, r.B, r.n, 1, e);
      if (off + need > ctx->arena_bytes) break;
      r.offset = off;
      r.slot = need;
      off += need;
      batch.push_back(r);
      idx.push_back(i1);
      ++i1;
    }
    if (batch.empty())
      return fail(ctx, PROTEA_ERR_OOM, "evaluate_round: client " + std::to_string(clients[i0].client_id) +
                                           ": evaluation slot exceeds the arena");
    ExecExtras xx;
    xx.eval = true;
    xx.shards = &ctx->val_shards;
    std::vector<double> st;
    xx.stats_out = &st;
    reset_ops(ctx, 0);
    protea_status s2 = execute(ctx, batch, wg, nullptr, 0.0f, 0, 0, 0, nullptr, nullptr, &xx);
    if (s2 != PROTEA_OK) return s2;
    for (size_t k = 0; k < batch.size(); ++k) {
      protea_eval_result& r = per_client[idx[k]];
      r.loss_sum = st[2 * k];
      r.correct = (uint64_t)llround(st[2 * k + 1]);
      r.n = (uint64_t)batch[k].n;
    }
    i0 = i1;
  }
  if (total) {
    std::memset(total, 0, sizeof(*total));
    for (size_t i = 0; i < n; ++i) {  // client order
      total->loss_sum += per_client[i].loss_sum;
      total->correct += per_client[i].correct;
      total->n += per_client[i].n;
    }
  }
  return PROTEA_OK;
}

static int64_t cnn_params(int q, int classes) {
  const int64_t C1 = 8 * q, C2 = 16 * q, F = 128 * q;
  return C1 * 75 + C1 + C2 * 25 * C1 + C2 + F * 64 * C2 + F + (int64_t)classes * F + classes;
}

protea_status protea_heterofl_extract(protea_ctx* ctx, int32_t classes, const float* global_full, int32_t width_q,
                                      float* sub_out) {
  if (!ctx) return PROTEA_ERR_INVALID;
  if (!global_full || !sub_out) return fail(ctx, PROTEA_ERR_INVALID, "heterofl_extract: null argument");
  if (classes < 2 || classes > 64) return fail(ctx, PROTEA_ERR_INVALID, "heterofl_extract: classes not in [2, 64]");
  if (width_q != 1 && width_q != 2 && width_q != 4)
    return fail(ctx, PROTEA_ERR_INVALID, "heterofl_extract: width_q not in {1, 2, 4}");
  CK(cudaSetDevice(ctx->device));
  const int64_t P = cnn_params(4, classes);
  k_heterofl_extract<<<grid_for(P, 256), 256, 0, ctx->stream>>>(global_full, width_q, classes, sub_out, P);
  ctx->launches++;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  return PROTEA_OK;
}

protea_status protea_heterofl_aggregate(protea_ctx* ctx, int32_t classes, const float* global_full,
                                        const float* const* params, const int32_t* width_q,
                                        const int64_t* num_examples, size_t n, float* out) {
  if (!ctx) return PROTEA_ERR_INVALID;
  if (n == 0) return fail(ctx, PROTEA_ERR_EMPTY, "heterofl_aggregate: no results to aggregate");
  if (!global_full || !params || !width_q || !num_examples || !out)
    return fail(ctx, PROTEA_ERR_INVALID, "heterofl_aggregate: null argument");
  if (classes < 2 || classes > 64) return fail(ctx, PROTEA_ERR_INVALID, "heterofl_aggregate: classes not in [2, 64]");
  std::vector<double> w(n);
  for (size_t k = 0; k < n; ++k) {
    const std::string who = "heterofl_aggregate: client " + std::to_string(k);
    if (!params[k]) return fail(ctx, PROTEA_ERR_INVALID, who + ": params is null");
    if (width_q[k] != 1 && width_q[k] != 2 && width_q[k] != 4)
      return fail(ctx, PROTEA_ERR_INVALID, who + ": width_q not in {1, 2, 4}");
    if (num_examples[k] <= 0) return fail(ctx, PROTEA_ERR_INVALID, who + ": num_examples <= 0");
    w[k] = (double)num_examples[k];
  }
  CK(cudaSetDevice(ctx->device));
  CK(ctx->ptrs.reserve(n));
  CK(ctx->wts.reserve(n));
  CK(ctx->wq.reserve(n));
  CK(cudaMemcpyAsync(ctx->ptrs.p, params, n * sizeof(float*), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->wts.p, w.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->wq.p, width_q, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  const int64_t P = cnn_params(4, classes);
  k_heterofl<<<grid_for(P, 256), 256, 0, ctx->stream>>>(ctx->ptrs.p, ctx->wq.p, ctx->wts.p, (int)n, global_full, out,
                                                         P, classes);
  ctx->launches++;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  return PROTEA_OK;
}

protea_status protea_fedavg(protea_ctx* ctx, const float* const* params, const int64_t* num_examples, size_t n,
                            size_t dim, float* out) {
  if (!ctx) return PROTEA_ERR_INVALID;
  if (n == 0) return fail(ctx, PROTEA_ERR_EMPTY, "fedavg: no results to aggregate");
  if (!params || !num_examples || !out || dim == 0) return fail(ctx, PROTEA_ERR_INVALID, "fedavg: null argument");
  int64_t N = 0;
  std::vector<double> w(n);
  for (size_t k = 0; k < n; ++k) {
    if (!params[k]) return fail(ctx, PROTEA_ERR_INVALID, "fedavg: params[" + std::to_string(k) + "] is null");
    if (num_examples[k] <= 0)
      return fail(ctx, PROTEA_ERR_INVALID, "fedavg: num_examples[" + std::to_string(k) + "] <= 0");
    N += num_examples[k];
    w[k] = (double)num_examples[k];
  }
  if (N == 0) return fail(ctx, PROTEA_ERR_ZERO_WEIGHT, "fedavg: zero total weight");
  CK(cudaSetDevice(ctx->device));
  CK(ctx->ptrs.reserve(n));
  CK(ctx->wts.reserve(n));
  CK(cudaMemcpyAsync(ctx->ptrs.p, params, n * sizeof(float*), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->wts.p, w.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
  k_fedavg<<<grid_for((int64_t)dim, 256), 256, 0, ctx->stream>>>(ctx->ptrs.p, ctx->wts.p, (int)n, (double)N, out,
                                                                 (int64_t)dim);
  ctx->launches++;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  return PROTEA_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// include/protea_selftest.h
// ---------------------------------------------------------------------------
extern "C" protea_status protea_selftest_gemm(const void* A, const void* B, float* D, int32_t M, int32_t N,
                                              int32_t K, int32_t mn_major) {
  if (!A || !B || !D || M <= 0 || M % 128 || N <= 0 || N > 64 || K <= 0 || K % 64) {
    set_global_error("selftest_gemm: need M % 128 == 0, 0 < N <= 64, K % 64 == 0, non-null pointers");
    return PROTEA_ERR_INVALID;
  }
  int h[2 + 4] = {0, M / 128, 0, 0, 1, 0};  // prefix[0..1], task {rec, step, rows, base}
  int* dtab = nullptr;
  if (cudaMalloc(&dtab, sizeof(h)) != cudaSuccess) return PROTEA_ERR_CUDA;
  cudaMemcpy(dtab, h, sizeof(h), cudaMemcpyHostToDevice);
  const Task* tasks = reinterpret_cast<const Task*>(dtab + 2);
  constexpr int SMEM = tc_smem_bytes<64, 4>();
  if (mn_major) {
    TcDenseMN op{nullptr, (const bf16*)A, (const bf16*)B, D, M, N, K};
    cudaFuncSetAttribute(k_gemm_tc<64, 4, TcDenseMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    k_gemm_tc<64, 4, TcDenseMN><<<M / 128, kTcThreads, SMEM>>>(op, tasks, dtab, 1);
  } else {
    TcDense op{nullptr, (const bf16*)A, (const bf16*)B, D, M, N, K};
    cudaFuncSetAttribute(k_gemm_tc<64, 4, TcDense>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    k_gemm_tc<64, 4, TcDense><<<M / 128, kTcThreads, SMEM>>>(op, tasks, dtab, 1);
  }
  cudaError_t e = cudaDeviceSynchronize();
  cudaFree(dtab);
  if (e != cudaSuccess) {
    set_global_error(std::string("selftest_gemm: ") + cudaGetErrorString(e));
    return PROTEA_ERR_CUDA;
  }
  return PROTEA_OK;
}
