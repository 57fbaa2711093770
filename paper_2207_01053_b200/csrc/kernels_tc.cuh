// kernels_tc.cuh — bf16 tensor-core (tcgen05 / TMEM) grouped GEMMs of one
// lock-step iteration (bf16 mode).
//
// Same grouped structure as kernels_simt.cuh (one launch per layer-op over every
// active client; CTA -> (client, tile) by binary search over a prefix table),
// but each CTA computes a 128 x BN output tile on the 5th-generation tensor
// cores: 8 producer warps stream 64-wide K blocks of both operands into a
// STAGES-deep shared-memory ring with 16-byte cp.async (the operands are
// implicit-GEMM gathers: im2col of NHWC activations, transposed weights, ...),
// one elected thread of warp 8 issues tcgen05.mma (M=128, N<=BN, K=16, bf16
// in, fp32 accumulate in TMEM) and tcgen05.commit releases each stage, then the
// 8 producer warps drain the accumulator with tcgen05.ld (warps w and w+4 share
// TMEM lanes 32(w%4).., splitting the columns) and run the layer's fused
// epilogue (bias+ReLU+2x2 pool / ReLU-mask + pool-backward scatter / SGD update
// of fp32 master + bf16 shadow weights).
//
// Each producer thread owns fixed (row, chunk) coordinates of the tile for
// the whole K loop, so the per-row part of the gather address (image, y, x,
// base pointer) is computed once per tile ("pre" states); per K block only the
// tap / channel offset changes.  Channel counts are compile-time (width WQ).
//
// Op sizes per client-step (rows = |beta|, CNN-w channels C1, C2, F; K1 = 64 C2):
//   conv2 fwd   M = rows*256 (quad-major) N = C2    K = 25 C1      A K-major, B K-major
//   conv2 dgrad M = rows*256              N = C1    K = 25 C2      A K-major, B MN-major
//   conv2 wgrad M = 25 C1 + 1 (bias row)  N = C2    K = rows*256   A MN-major, B MN-major
//   fc1 fwd     M = F                     N = rows  K = K1         A K-major, B K-major
//   fc1 dgrad   M = K1                    N = rows  K = F          A MN-major, B K-major
//   fc1 wgrad   M = K1                    N = F     K = rows       A MN-major, B MN-major
#pragma once
#include "device.cuh"
#include "kernels_simt.cuh"
#include "tc.cuh"

namespace protea {

typedef __nv_bfloat16 bf16;

struct TcTile {
  const ClientRec* c;
  Task tk;
  int m0, n0;
  int nk;     // 64-wide K blocks
  int n_mma;  // instruction N (multiple of 16, <= BN)
};

__device__ __align__(16) const uint16_t kOneChunk[8] = {0x3F80, 0, 0, 0, 0, 0, 0, 0};  // bf16 {1,0,...,0}

constexpr int kTcProd = 256;               // producer / epilogue threads (8 warps)
constexpr int kTcThreads = kTcProd + 32;   // + the MMA warp

template <bool MN, int R>
__device__ __forceinline__ void chunk_coords(int q, int& i, int& j) {
  if (MN) {  // i = k row in [0,64), j = mn group in [0, R/8)
    i = (q / R) * 8 + (q & 7);
    j = (q >> 3) % (R / 8);
  } else {  // i = mn row in [0, R), j = k chunk in [0, 8)
    i = (q >> 6) * 8 + (q & 7);
    j = (q >> 3) & 7;
  }
}

template <int BN, int STAGES>
constexpr int tc_smem_bytes() {  // + 1 KB to realign the dynamic window to 1024 B (128-byte-swizzle atoms)
  return STAGES * (128 * 64 * 2 + BN * 64 * 2) + (2 * STAGES + 1) * 8 + 16 + 1024;
}

// Default UMMA descriptors of the cp.async layouts (see tc.cuh).
template <bool MN, int R>
__device__ __forceinline__ uint64_t cp_desc(uint32_t base, int ks) {
  return MN ? tc::sdesc(base + 32 * R * ks, 16 * R, 128) : tc::sdesc(base + 256 * ks, 128, 1024);
}
template <class Op>
struct has_tma {
  template <class U>
  static constexpr bool f(decltype(U::TMA)*) { return U::TMA; }
  template <class U>
  static constexpr bool f(...) { return false; }
  static constexpr bool value = f<Op>(nullptr);
};

template <class Op>
struct has_finish {
  template <class U>
  static constexpr bool f(decltype(U::FINISH)*) { return U::FINISH; }
  template <class U>
  static constexpr bool f(...) { return false; }
  static constexpr bool value = f<Op>(nullptr);
};

template <class Op>
struct has_pfinish {
  template <class U>
  static constexpr bool f(decltype(U::PFINISH)*) { return U::PFINISH; }
  template <class U>
  static constexpr bool f(...) { return false; }
  static constexpr bool value = f<Op>(nullptr);
};

template <class Op>
struct has_block_epi {  // the op drains the whole TMEM tile itself (all 8 epilogue warps, shared memory)
  template <class U>
  static constexpr bool f(decltype(U::BLOCK_EPI)*) { return U::BLOCK_EPI; }
  template <class U>
  static constexpr bool f(...) { return false; }
  static constexpr bool value = f<Op>(nullptr);
};

template <class Op>
struct min_blocks {  // resident CTAs per SM the op is compiled for (register cap), default 1
  template <class U>
  static constexpr int f(decltype(U::MIN_BLOCKS)*) { return U::MIN_BLOCKS; }
  template <class U>
  static constexpr int f(...) { return 1; }
  static constexpr int value = f<Op>(nullptr);
};

template <class Op>
struct has_ksteps {  // the op's single K block holds fewer than 4 MMA K steps (Op::KSTEPS + op.ksteps(t))
  template <class U>
  static constexpr bool f(decltype(U::KSTEPS)*) { return U::KSTEPS; }
  template <class U>
  static constexpr bool f(...) { return false; }
  static constexpr bool value = f<Op>(nullptr);
};

template <class Op>
struct halo_stages {  // depth of k_conv_persistent's halo ring (Op::HSTAGES), default 2
  template <class U>
  static constexpr int f(decltype(U::HSTAGES)*) { return U::HSTAGES; }
  template <class U>
  static constexpr int f(...) { return 2; }
  static constexpr int value = f<Op>(nullptr);
};

template <int BN, int STAGES, class Op>
__global__ void __launch_bounds__(kTcThreads, min_blocks<Op>::value)
    k_gemm_tc(const Op op, const Task* __restrict__ tasks, const int* __restrict__ prefix, int ntask) {
  constexpr bool TMA = has_tma<Op>::value;
  constexpr int A_BYTES = 128 * 64 * 2, B_BYTES = BN * 64 * 2, STAGE = A_BYTES + B_BYTES;
  constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  constexpr int LAG = (STAGES - 1) < 2 ? (STAGES - 1) : 2;  // STAGES == 1: single-K-block ops (LAG 0)
  constexpr int NA = 1024 / kTcProd;                             // A chunks per producer thread
  constexpr int NB = (BN * 8 + kTcProd - 1) / kTcProd;           // B chunks per producer thread
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int ti = find_task(prefix, ntask, blockIdx.x);
  TcTile t;
  t.tk = tasks[ti];
  t.c = op.recs + t.tk.rec;
  op.setup(t, blockIdx.x - __ldg(prefix + ti));
  const uint64_t t_start = threadIdx.x == 0 ? globaltimer() : 0;

  const uint32_t bar0 = tc::smem_u32(bars);
  const uint32_t done = bar0 + 16 * STAGES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(bar0 + 8 * s, TMA ? 1 : kTcProd);  // full[s]: TMA expect_tx, or one arrive per producer
      tc::mbar_init(bar0 + 8 * (STAGES + s), 1);    // empty[s]: tcgen05.commit
    }
    tc::mbar_init(done, 1);
    tc::mbar_fence_init();
  }
  if (warp == 8) tc::tmem_alloc(tc::smem_u32(tmem_slot), TMEM_COLS);
  const uint32_t sbase = tc::smem_u32(smem);
  if constexpr (TMA) {
    if (warp < 8) {  // constant operand groups (e.g. the bias "ones" row), written once into every stage
      for (int s = 0; s < STAGES; ++s) op.init_stage(t, smem + s * STAGE, smem + s * STAGE + A_BYTES);
      tc::fence_proxy_async();
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();

  if constexpr (TMA) {
    if (warp == 0 && lane == 0) {
      // ---------------- TMA producer (one thread)
      for (int kb = 0; kb < t.nk; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) tc::mbar_wait(bar0 + 8 * (STAGES + s), ((kb / STAGES) - 1) & 1);
        const uint32_t a_base = sbase + s * STAGE, b_base = a_base + A_BYTES;
        tc::mbar_expect_tx(bar0 + 8 * s, op.tx_bytes(t, kb));
        op.tma_issue(t, kb, a_base, b_base, bar0 + 8 * s);
      }
    }
  }
  if (warp < 8) {
    // ---------------- cp.async producers
    if constexpr (!TMA) {
    const int tid = threadIdx.x;
    const void* any = op.any(t);
    typename Op::PA pa[NA];
    typename Op::PB pb[NB];
#pragma unroll
    for (int u = 0; u < NA; ++u) {
      int i, j;
      chunk_coords<Op::A_MN, 128>(tid + kTcProd * u, i, j);
      pa[u] = op.a_pre(t, i, j);
    }
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      int i = 0, j = 0;
      if (tid + kTcProd * u < BN * 8) chunk_coords<Op::B_MN, BN>(tid + kTcProd * u, i, j);
      pb[u] = op.b_pre(t, i, j);
    }
    for (int kb = 0; kb < t.nk; ++kb) {
      const int s = kb % STAGES;
      if (kb >= STAGES) tc::mbar_wait(bar0 + 8 * (STAGES + s), ((kb / STAGES) - 1) & 1);
      const uint32_t a_base = sbase + s * STAGE, b_base = a_base + A_BYTES;
#pragma unroll
      for (int u = 0; u < NA; ++u) tc::cp16(a_base + 16 * (tid + kTcProd * u), op.a_src(t, pa[u], kb), any);
#pragma unroll
      for (int u = 0; u < NB; ++u)
        if (tid + kTcProd * u < BN * 8) tc::cp16(b_base + 16 * (tid + kTcProd * u), op.b_src(t, pb[u], kb), any);
      tc::cp_commit();
      if (kb >= LAG) {
        tc::cp_wait<LAG>();
        tc::fence_proxy_async();
        tc::mbar_arrive(bar0 + 8 * ((kb - LAG) % STAGES));
      }
    }
    tc::cp_wait<0>();
    tc::fence_proxy_async();
    for (int kb = (t.nk - LAG > 0 ? t.nk - LAG : 0); kb < t.nk; ++kb) tc::mbar_arrive(bar0 + 8 * (kb % STAGES));
    }

    // ---------------- epilogue: TMEM -> registers -> fused layer epilogue
    if constexpr (has_block_epi<Op>::value) {
      op.block_epilogue(t, smem, tmem, warp, lane, done);  // waits for the MMAs itself (after its first loads)
    } else {
      tc::mbar_wait(done, 0);
      tc::fence_after();
      const int row = (warp & 3) * 32 + lane;
      for (int c0 = (warp >> 2) * 16; c0 < t.n_mma; c0 += 32) {
        float v[16];
        tc::tmem_ld16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0, v);
        op.epilogue(t, row, c0, v);
      }
    }
  } else {
    // ---------------- MMA issuer (warp 8, elected lane issues)
    {
      const uint32_t idesc = tc::idesc_bf16(128, t.n_mma, Op::A_MN, Op::B_MN);
      // descriptors are linear in the stage base and the k step: precompute, then add constants
      uint64_t da0, dak, db0, dbk;
      if constexpr (TMA) {
        da0 = op.a_desc(t, sbase, 0);
        dak = op.a_desc(t, sbase, 1) - da0;
        db0 = op.b_desc(t, sbase + A_BYTES, 0);
        dbk = op.b_desc(t, sbase + A_BYTES, 1) - db0;
      } else {
        da0 = cp_desc<Op::A_MN, 128>(sbase, 0);
        dak = cp_desc<Op::A_MN, 128>(sbase, 1) - da0;
        db0 = cp_desc<Op::B_MN, BN>(sbase + A_BYTES, 0);
        dbk = cp_desc<Op::B_MN, BN>(sbase + A_BYTES, 1) - db0;
      }
      for (int kb = 0; kb < t.nk; ++kb) {
        const int s = kb % STAGES;
        tc::mbar_wait(bar0 + 8 * s, (kb / STAGES) & 1);
        tc::fence_after();
        const uint64_t so = (uint64_t)(s * (STAGE >> 4));
        int nks = 4;
        if constexpr (has_ksteps<Op>::value) nks = op.ksteps(t);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          if (ks < nks) tc::mma_bf16_w(tmem, da0 + so + ks * dak, db0 + so + ks * dbk, idesc, (kb | ks) != 0);
        tc::commit_w(bar0 + 8 * (STAGES + s));
      }
      tc::commit_w(done);
    }
    __syncwarp();
  }
  pdl_trigger();  // main work done: let the next kernel's CTAs start on the SMs this grid frees
  tc::fence_before();
  __syncthreads();
  if (warp == 8) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, TMEM_COLS);
  }
  if constexpr (has_finish<Op>::value) op.finish(t);  // e.g. last split-K CTA reduces and updates
  if (threadIdx.x == 0 && op.recs && t.c->sm_ns)  // K9: per-client SM-time attribution (CTA duration)
    atomicAdd((unsigned long long*)t.c->sm_ns, (unsigned long long)(globaltimer() - t_start));
}

// --------------------------------------------------------------------------
// Persistent variant for TMA ops without split-K finish (fc1 fwd / dgrad): a CTA
// walks a contiguous range of the launch's tiles; warp 9 streams every tile's K
// blocks through the STAGES ring, warp 8 issues the MMAs into one of two TMEM
// accumulators, warps 0-7 drain the other one through the op's epilogue, so the
// epilogue of tile i overlaps the loads and MMAs of tile i+1 (the per-CTA
// prologue / drain / epilogue serialisation of k_gemm_tc was the bottleneck).
// --------------------------------------------------------------------------
constexpr int kPersThreads = 320;
template <int BN, int STAGES>
constexpr int pers_smem_bytes() {
  return STAGES * (128 * 64 * 2 + BN * 64 * 2) + (2 * STAGES + 4) * 8 + 16 + 1024;
}
template <int BN, int STAGES, class Op>
__global__ void __launch_bounds__(kPersThreads, 1)
    k_gemm_persistent(const Op op, const Task* __restrict__ tasks, const int* __restrict__ prefix, int ntask) {
  static_assert(has_tma<Op>::value && !has_finish<Op>::value, "persistent GEMM: TMA ops without finish");
  constexpr int A_BYTES = 128 * 64 * 2, B_BYTES = BN * 64 * 2, STAGE = A_BYTES + B_BYTES;
  constexpr int TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 256;
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
      tc::mbar_init(full + 8 * s, 1);
      tc::mbar_init(empty + 8 * s, 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(acc_full + 8 * i, 1);
      tc::mbar_init(acc_empty + 8 * i, 8);
    }
    tc::mbar_fence_init();
  }
  if (warp == 8) tc::tmem_alloc(tc::smem_u32(tmem_slot), TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = tc::smem_u32(smem);
  TcTile t;
  TaskCursor cur;
  cur.init(prefix, ntask, g0 < total ? g0 : total - 1);
  pdl_wait();
  if (warp == 9) {
    if (lane == 0) {  // ---------------- TMA producer
      int it = 0;
      for (int g = g0; g < g1; ++g) {
        if (cur.advance(prefix, g) || g == g0) {
          t.tk = tasks[cur.ti];
          t.c = op.recs + t.tk.rec;
        }
        op.setup(t, g - cur.lo);
        for (int kb = 0; kb < t.nk; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) tc::mbar_wait(empty + 8 * s, ((it / STAGES) - 1) & 1);
          const uint32_t a_base = sbase + s * STAGE;
          tc::mbar_expect_tx(full + 8 * s, op.tx_bytes(t, kb));
          op.tma_issue(t, kb, a_base, a_base + A_BYTES, full + 8 * s);
        }
      }
    }
  } else if (warp == 8) {
    if (g0 < g1) {  // ---------------- MMA issuer (whole warp, elected lane issues)
      t.tk = tasks[cur.ti];
      t.c = op.recs + t.tk.rec;
      const uint64_t da0 = op.a_desc(t, sbase, 0), dak = op.a_desc(t, sbase, 1) - da0;
      const uint64_t db0 = op.b_desc(t, sbase + A_BYTES, 0), dbk = op.b_desc(t, sbase + A_BYTES, 1) - db0;
      int it = 0, i = 0;
      for (int g = g0; g < g1; ++g, ++i) {
        if (cur.advance(prefix, g)) {
          t.tk = tasks[cur.ti];
          t.c = op.recs + t.tk.rec;
        }
        op.setup(t, g - cur.lo);
        const uint32_t idesc = tc::idesc_bf16(128, t.n_mma, Op::A_MN, Op::B_MN);
        const int acc = i & 1;
        if (i >= 2) tc::mbar_wait(acc_empty + 8 * acc, ((i >> 1) - 1) & 1);
        tc::fence_after();
        const uint32_t dt = tmem + acc * BN;
        for (int kb = 0; kb < t.nk; ++kb, ++it) {
          const int s = it % STAGES;
          tc::mbar_wait(full + 8 * s, (it / STAGES) & 1);
          tc::fence_after();
          const uint64_t so = (uint64_t)(s * (STAGE >> 4));
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            tc::mma_bf16_w(dt, da0 + so + ks * dak, db0 + so + ks * dbk, idesc, (kb | ks) != 0);
          tc::commit_w(empty + 8 * s);
        }
        tc::commit_w(acc_full + 8 * acc);
      }
    }
    __syncwarp();
  } else {  // ---------------- epilogue warps 0-7
    const int row = (warp & 3) * 32 + lane;
    int i = 0;
    for (int g = g0; g < g1; ++g, ++i) {
      if (cur.advance(prefix, g) || g == g0) {
        t.tk = tasks[cur.ti];
        t.c = op.recs + t.tk.rec;
      }
      op.setup(t, g - cur.lo);
      const int acc = i & 1;
      tc::mbar_wait(acc_full + 8 * acc, (i >> 1) & 1);
      tc::fence_after();
      for (int c0 = (warp >> 2) * 16; c0 < t.n_mma; c0 += 32) {
        float v[16];
        tc::tmem_ld16(tmem + acc * BN + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0, v);
        op.epilogue(t, row, c0, v);
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(acc_empty + 8 * acc);
      if constexpr (has_pfinish<Op>::value) op.pfinish(t);  // split-K: the last split reduces (epilogue warps)
    }
  }
  pdl_trigger();  // main work done: let the next kernel's CTAs start on the SMs this grid frees
  tc::fence_before();
  __syncthreads();
  if (warp == 8) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, TMEM_COLS);
  }
  if (threadIdx.x == 0 && g1 > g0) {  // K9: split the CTA's duration over its clients by tile count
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

__device__ __forceinline__ int round16(int x) { return (x + 15) & ~15; }

// Vectorised epilogue helpers: a thread owns 16 consecutive channels of one pixel.
template <int N>  // N = 8 or 16 bf16
__device__ __forceinline__ void st_bf16(bf16* dst, const float* v) {
  uint32_t w[N / 2];
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    w[i] = *reinterpret_cast<const uint32_t*>(&h);
  }
  reinterpret_cast<uint4*>(dst)[0] = make_uint4(w[0], w[1], w[2], w[3]);
  if (N == 16) reinterpret_cast<uint4*>(dst)[1] = make_uint4(w[4], w[5], w[6], w[7]);
}
template <int N>
__device__ __forceinline__ void ld_bf16(const bf16* src, float* v) {
  uint4 q[2];
  q[0] = reinterpret_cast<const uint4*>(src)[0];
  if (N == 16) q[1] = reinterpret_cast<const uint4*>(src)[1];
  const uint32_t* w = reinterpret_cast<const uint32_t*>(q);
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
    v[2 * i] = __low2float(h);
    v[2 * i + 1] = __high2float(h);
  }
}
template <int N>
__device__ __forceinline__ void st_u8(uint8_t* dst, const int* a) {
  uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < N; ++i) w[i >> 2] |= (uint32_t)a[i] << (8 * (i & 3));
  if (N == 16)
    *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
  else
    *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
}
template <int N>
__device__ __forceinline__ void ld_u8(const uint8_t* src, int* a) {
  uint32_t w[4];
  if (N == 16) {
    const uint4 q = *reinterpret_cast<const uint4*>(src);
    w[0] = q.x, w[1] = q.y, w[2] = q.z, w[3] = q.w;
  } else {
    const uint2 q = *reinterpret_cast<const uint2*>(src);
    w[0] = q.x, w[1] = q.y;
  }
#pragma unroll
  for (int i = 0; i < N; ++i) a[i] = (w[i >> 2] >> (8 * (i & 3))) & 0xFF;
}

// 2x2 max-pool of a warp's 16 columns: values of the 4 window lanes (q order
// (0,0),(0,1),(1,0),(1,1)), first maximum wins (strict >); result in the writer lane.
__device__ __forceinline__ void pool_lanes(const float (&val)[16], int l0, int l1, int l2, int l3, float (&best)[16],
                                           int (&arg)[16]) {
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const float v0 = __shfl_sync(0xffffffffu, val[j], l0), v1 = __shfl_sync(0xffffffffu, val[j], l1);
    const float v2 = __shfl_sync(0xffffffffu, val[j], l2), v3 = __shfl_sync(0xffffffffu, val[j], l3);
    float b = v0;
    int a = 0;
    if (v1 > b) { b = v1; a = 1; }
    if (v2 > b) { b = v2; a = 2; }
    if (v3 > b) { b = v3; a = 3; }
    best[j] = b;
    arg[j] = a;
  }
}

// compile-time CNN-w channel counts for width WQ/4
template <int WQ>
struct CnnW {
  static constexpr int C1 = 8 * WQ, C2 = 16 * WQ, F = 128 * WQ, K1 = 64 * C2;
  static constexpr int L1 = WQ == 1 ? 3 : WQ == 2 ? 4 : 5;  // log2 C1
  static constexpr int L2 = L1 + 1;                          // log2 C2
};

// --------------------------------------------------------------------------
// CNN ops on tensor cores (bf16 activations, bf16 shadow weights B_WSH)
// --------------------------------------------------------------------------
template <int WQ>
struct TcConv2Wgrad {  // full reduction in one CTA -> SGD update in the epilogue (no split-K partials)
  typedef CnnW<WQ> W;
  static constexpr bool A_MN = true, B_MN = true;
  struct PA { int i, dy, dx, ci, kind; };  // kind 0: gather, 1: bias ones row, 2: zero
  struct PB { int i, n0; };
  const ClientRec* recs;
  CnnDims d;
  float lr;
  __device__ void setup(TcTile& t, int local) const {
    t.m0 = local * 128;
    t.n0 = 0;
    t.nk = t.tk.rows * 4;  // rows*256 pixels / 64
    t.n_mma = W::C2 < 16 ? 16 : W::C2;
  }
  __device__ const void* any(const TcTile& t) const { return t.c->params; }
  __device__ PA a_pre(const TcTile& t, int i, int j) const {
    const int mg = t.m0 + 8 * j, Kw = 25 * W::C1;
    if (mg == Kw) return PA{i, 0, 0, 0, 1};
    if (mg > Kw) return PA{i, 0, 0, 0, 2};
    const int tap = mg >> W::L1, ky = tap / 5, kx = tap - ky * 5;
    return PA{i, ky - 2, kx - 2, mg & (W::C1 - 1), 0};
  }
  __device__ const void* a_src(const TcTile& t, const PA& s, int kb) const {
    if (s.kind) return s.kind == 1 ? (const void*)kOneChunk : nullptr;
    const int p = kb * 64 + s.i, r = p >> 8, sy = ((p >> 4) & 15) + s.dy, sx = (p & 15) + s.dx;
    if ((unsigned)sy >= 16u || (unsigned)sx >= 16u) return nullptr;
    return (const bf16*)t.c->buf[B_A1] + ((int64_t)r * 256 + sy * 16 + sx) * W::C1 + s.ci;
  }
  __device__ PB b_pre(const TcTile& t, int i, int j) const { return PB{i, 8 * j}; }
  __device__ const void* b_src(const TcTile& t, const PB& s, int kb) const {
    if (s.n0 >= W::C2) return nullptr;
    return (const bf16*)t.c->buf[B_DZ2] + (int64_t)(kb * 64 + s.i) * W::C2 + s.n0;
  }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
    const int m = t.m0 + row, Kw = 25 * W::C1;
    if (m > Kw) return;
    float* P = t.c->params;
    bf16* S = (bf16*)t.c->buf[B_WSH];
    if (m == Kw) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (c0 + j < W::C2) P[d.b2 + c0 + j] -= lr * v[j];
      return;
    }
    float w[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) w[j] = c0 + j < W::C2 ? P[d.w2 + (int64_t)(c0 + j) * Kw + m] : 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (c0 + j < W::C2) {
        const int64_t idx = d.w2 + (int64_t)(c0 + j) * Kw + m;
        const float nw = w[j] - lr * v[j];
        P[idx] = nw;
        S[idx] = __float2bfloat16_rn(nw);
      }
  }
};

template <int WQ>
struct TcFc1Fwd {
  typedef CnnW<WQ> W;
  static constexpr bool A_MN = false, B_MN = false;
  struct PA { const bf16* p; };
  struct PB { const bf16* p; };
  const ClientRec* recs;
  CnnDims d;
  __device__ void setup(TcTile& t, int local) const {
    t.m0 = local * 128;
    t.n0 = 0;
    t.nk = W::K1 / 64;
    t.n_mma = round16(t.tk.rows);
  }
  __device__ const void* any(const TcTile& t) const { return t.c->params; }
  __device__ PA a_pre(const TcTile& t, int i, int j) const {
    return PA{reinterpret_cast<const bf16*>(t.c->params + d.w3) + (int64_t)(t.m0 + i) * W::K1 + 8 * j};  // hi plane
  }
  __device__ const void* a_src(const TcTile& t, const PA& s, int kb) const { return s.p + kb * 64; }
  __device__ PB b_pre(const TcTile& t, int i, int j) const {
    return PB{i < t.tk.rows ? (const bf16*)t.c->buf[B_A2] + (int64_t)i * W::K1 + 8 * j : nullptr};
  }
  __device__ const void* b_src(const TcTile& t, const PB& s, int kb) const { return s.p ? s.p + kb * 64 : nullptr; }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
    const int f = t.m0 + row;
    const float* params = reinterpret_cast<const float*>(__ldg(reinterpret_cast<const unsigned long long*>(&t.c->params)));
    bf16* h = reinterpret_cast<bf16*>(__ldg(reinterpret_cast<const unsigned long long*>(t.c->buf) + B_H));
    const float b = params[d.b3 + f];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int r = c0 + j;
      if (r < t.tk.rows) h[(int64_t)r * W::F + f] = __float2bfloat16_rn(fmaxf(v[j] + b, 0.f));
    }
  }
};

template <int WQ>
struct TcFc1Dgrad {
  typedef CnnW<WQ> W;
  static constexpr bool A_MN = true, B_MN = false;
  struct PA { const bf16* p; };
  struct PB { const bf16* p; };
  const ClientRec* recs;
  CnnDims d;
  __device__ void setup(TcTile& t, int local) const {
    t.m0 = local * 128;
    t.n0 = 0;
    t.nk = W::F / 64;
    t.n_mma = round16(t.tk.rows);
  }
  __device__ const void* any(const TcTile& t) const { return t.c->params; }
  __device__ PA a_pre(const TcTile& t, int i, int j) const {
    return PA{reinterpret_cast<const bf16*>(t.c->params + d.w3) + (int64_t)i * W::K1 + t.m0 + 8 * j};  // hi plane
  }
  __device__ const void* a_src(const TcTile& t, const PA& s, int kb) const { return s.p + (int64_t)kb * 64 * W::K1; }
  __device__ PB b_pre(const TcTile& t, int i, int j) const {
    return PB{i < t.tk.rows ? (const bf16*)t.c->buf[B_DH] + (int64_t)i * W::F + 8 * j : nullptr};
  }
  __device__ const void* b_src(const TcTile& t, const PB& s, int kb) const { return s.p ? s.p + kb * 64 : nullptr; }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
    const int n1 = t.m0 + row;
    const int p = n1 >> W::L2, c = n1 & (W::C2 - 1), py = p >> 3, px = p & 7;
    // the three buffer pointers together, read-only path (a dz2 pointer load issued after the mask loads was
    // the kernel's top stall: 27 % of warp samples, ncu)
    const unsigned long long* bufs = reinterpret_cast<const unsigned long long*>(t.c->buf);
    const unsigned long long u_a2 = __ldg(bufs + B_A2), u_i2 = __ldg(bufs + B_I2), u_dz = __ldg(bufs + B_DZ2);
    const bf16* __restrict__ a2 = reinterpret_cast<const bf16*>(u_a2);
    const uint8_t* __restrict__ i2 = reinterpret_cast<const uint8_t*>(u_i2);
    bf16* __restrict__ dz2 = reinterpret_cast<bf16*>(u_dz);
    const int nr = t.tk.rows - c0;
    bf16 am[16];
    uint8_t ar[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {  // all mask / argmax loads in flight before the first store
      const int64_t o = (int64_t)(c0 + j) * W::K1 + n1;
      am[j] = j < nr ? __ldg(a2 + o) : __float2bfloat16_rn(0.f);
      ar[j] = j < nr ? __ldg(i2 + o) : 0;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j >= nr) continue;
      const int r = c0 + j;
      const float val = __bfloat162float(am[j]) > 0.f ? v[j] : 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int y = 2 * py + (q >> 1), x = 2 * px + (q & 1);
        dz2[((int64_t)r * 256 + y * 16 + x) * W::C2 + c] = __float2bfloat16_rn(q == ar[j] ? val : 0.f);
      }
    }
  }
};

template <int WQ>
struct TcFc1Wgrad {  // M = K1 (input features), N = F (outputs), K = rows; W <- W - lr dW
  typedef CnnW<WQ> W;
  static constexpr bool A_MN = true, B_MN = true;
  static constexpr int NT = 128;  // N tile (TMEM 128 columns -> up to 4 CTAs per SM)
  struct PA { const bf16* p; };
  struct PB { const bf16* p; };
  const ClientRec* recs;
  CnnDims d;
  float lr;
  __device__ void setup(TcTile& t, int local) const {
    const int nt = (W::F + NT - 1) / NT;
    t.m0 = (local / nt) * 128;
    t.n0 = (local % nt) * NT;
    t.nk = 1;  // rows <= 64
    t.n_mma = W::F - t.n0 < NT ? W::F - t.n0 : NT;
  }
  __device__ const void* any(const TcTile& t) const { return t.c->params; }
  __device__ PA a_pre(const TcTile& t, int i, int j) const {
    return PA{i < t.tk.rows ? (const bf16*)t.c->buf[B_A2] + (int64_t)i * W::K1 + t.m0 + 8 * j : nullptr};
  }
  __device__ const void* a_src(const TcTile& t, const PA& s, int kb) const { return s.p; }
  __device__ PB b_pre(const TcTile& t, int i, int j) const {
    const int n = t.n0 + 8 * j;
    return PB{i < t.tk.rows && n < W::F ? (const bf16*)t.c->buf[B_DH] + (int64_t)i * W::F + n : nullptr};
  }
  __device__ const void* b_src(const TcTile& t, const PB& s, int kb) const { return s.p; }
  // SGD on the fp32 master held as split planes (device.cuh): read hi + lo (4 B), write hi + lo (4 B) —
  // exactly SURVEY §8(d)'s 8 B per weight per client-step; the new hi plane is next step's operand.
  // A tile column (output f, the tile's 128 k1) is one 128-block of the layout: 256 B of upper halves and the
  // 256 B of lower halves right after them.  The 8 epilogue warps drain the tile 32 columns per pass through
  // shared memory (the free operand stage): coalesced 8-byte loads (one warp = one column = 2 x 256 B), each
  // thread updates its TMEM row's 16 columns in shared memory, coalesced 8-byte stores.
  static constexpr bool BLOCK_EPI = true;
  static constexpr int MIN_BLOCKS = 4;  // HBM-bound: 4 CTAs per SM (<= 56 registers)
  // Software-pipelined over passes of 32 columns: the first pass's weights are loaded before the MMAs are
  // waited for, and pass p + 1's loads are in flight while pass p is updated in shared memory (two 16 KB
  // staging buffers in the free operand stage).
  __device__ void block_epilogue(const TcTile& t, uint8_t* smem, uint32_t tmem, int warp, int lane,
                                 uint32_t done) const {
    uint16_t* Hp = reinterpret_cast<uint16_t*>(t.c->params + d.w3) + (t.m0 >> 7) * 256;  // this tile's k1 block
    uint16_t* Lp = Hp + 128;
    const int row = (warp & 3) * 32 + lane, cl = (warp >> 2) * 16;
    uint2 h[4], l[4];
    auto load = [&](int cb) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t o = (int64_t)(t.n0 + cb + 4 * warp + i) * 2 * W::K1 + 4 * lane;
        h[i] = *reinterpret_cast<const uint2*>(Hp + o);
        l[i] = *reinterpret_cast<const uint2*>(Lp + o);
      }
    };
    load(0);
    tc::mbar_wait(done, 0);
    tc::fence_after();
    // the staging buffer holds each weight as its fp32 value (hi/lo halves interleaved with byte permutes):
    // the update pass is one conflict-free 4-byte load and store per weight instead of two 2-byte of each
    for (int cb = 0, buf = 0; cb < t.n_mma; cb += 32, buf ^= 1) {
      uint32_t* sf = reinterpret_cast<uint32_t*>(smem) + buf * 4096;  // [32 columns][128 rows] fp32
#pragma unroll
      for (int i = 0; i < 4; ++i)
        *reinterpret_cast<uint4*>(sf + (4 * warp + i) * 128 + 4 * lane) =
            make_uint4(__byte_perm(l[i].x, h[i].x, 0x5410), __byte_perm(l[i].x, h[i].x, 0x7632),
                       __byte_perm(l[i].y, h[i].y, 0x5410), __byte_perm(l[i].y, h[i].y, 0x7632));
      if (cb + 32 < t.n_mma) load(cb + 32);
      asm volatile("bar.sync 1, 256;" ::: "memory");
      float v[16];
      tc::tmem_ld16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(cb + cl), v);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float* w = reinterpret_cast<float*>(sf) + (cl + j) * 128 + row;
        *w = *w - lr * v[j];  // (= split_join(hi, lo) - lr * g, stored back as its two halves below)
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t o = (int64_t)(t.n0 + cb + 4 * warp + i) * 2 * W::K1 + 4 * lane;
        const uint4 q = *reinterpret_cast<const uint4*>(sf + (4 * warp + i) * 128 + 4 * lane);
        *reinterpret_cast<uint2*>(Hp + o) = make_uint2(__byte_perm(q.x, q.y, 0x7632), __byte_perm(q.z, q.w, 0x7632));
        *reinterpret_cast<uint2*>(Lp + o) = make_uint2(__byte_perm(q.x, q.y, 0x5410), __byte_perm(q.z, q.w, 0x5410));
      }
    }
  }
  __device__ void epilogue(const TcTile&, int, int, const float (&)[16]) const {}
};

// --------------------------------------------------------------------------
// TMA-fed ops.  Operand tiles are loaded by the Tensor Memory Accelerator from
// per-client tensor maps (built on the host per slot, kept in global memory):
// every box is "8 channels x R rows" of 16-byte rows, which lands in shared
// memory as R consecutive 16-byte rows = UMMA canonical core matrices; conv
// halos (zero padding) are the TMA's out-of-bounds zero fill.  This bypasses
// L1 (the cp.async gathers above were L1TEX-throughput bound) and leaves one
// thread issuing ~16-24 bulk copies per 64-wide K block.
// --------------------------------------------------------------------------
enum TmapId : int {
  TM_A1 = 0,   // a1  [B][16][16][C1] box (8,16,8,1)   conv2 fwd A
  TM_A1W,      // a1                box (8,16,4,1)   conv2 wgrad A
  TM_DZ2W,     // dz2               box (8,16,4,1)   conv2 wgrad B
  TM_W2F,      // W2 shadow (25C1, C2)   box (8, C2) conv2 fwd B
  TM_W2D,      // W2 shadow (C1, 25, C2) box (8,1,C2) conv2 dgrad B
  TM_W3K,      // W3 shadow (K1, F)      box (64,128) 128B-swizzled, fc1 fwd A
  TM_W3M,      // W3 shadow (K1, F)      box (64,64)  128B-swizzled, fc1 dgrad A (MN-major)
  TM_A2,       // a2 (K1, B)             box (64,R)   128B-swizzled, fc1 fwd B
  TM_DH,       // dh (F, B)              box (64,R)   128B-swizzled, fc1 dgrad B
  TM_A1H,      // a1                box (8,16,12,1)  conv2 fwd halo (kernels_conv.cuh)
  TM_DZ2H,     // dz2               box (8,16,12,1)  conv2 dgrad halo
  TM_XSH,      // xs [B][36 Y][2 par][18 X' x 8] box (80,2,36,1)  conv1 fwd halo (kernels_conv.cuh)
  TM_XSW,      // xs                box (64,1,36,1)  conv1 wgrad: one x-shifted copy per dx
  TM_G,        // g1 [B][16][16][4 q][C1] box (64,8,16,1) 128B-swizzled  conv1 wgrad A (MN-major)
  TM_A1Q,      // a1  box (32,12,20,1) 64B-swizzled   conv2 wgrad single halo (width 1)
  TM_DZ2Q,     // dz2 box (64,8,16,1)  128B-swizzled  conv2 wgrad B, one image half (width 1)
  TM_DZ2Q1,    // dz2 box (32,12,20,1) 64B-swizzled   conv2 dgrad single halo, one 32-channel group (width 1)
  TM_W2FS,     // W2 shadow (800, 64)    box (64,64) 128B-swizzled  conv2 fwd weights (width 1)
  TM_W2DS,     // W2 shadow (32, 25, 64) box (32,1,64) 64B-swizzled conv2 dgrad weights (width 1)
  TM_COUNT
};
constexpr int kTmapSlots = 28;  // per-client map array (CNN: TmapId; ResNet-8: RTmapId, kernels_resnet_halo.cuh)
static_assert((int)TM_COUNT <= kTmapSlots, "CNN maps exceed the per-client map array");

__device__ __forceinline__ const void* tmap_of(const TcTile& t, int id) {
  return reinterpret_cast<const uint8_t*>(t.c->tmaps) + 128 * id;
}

template <int WQ>
struct TmaConv2Fwd {  // M = rows*256 (natural order, tile = 8 image rows), N = C2, K = 25 C1
  typedef CnnW<WQ> W;
  static constexpr bool TMA = true, A_MN = false, B_MN = false;
  const ClientRec* recs;
  CnnDims d;
  __device__ void setup(TcTile& t, int local) const {
    t.m0 = local * 128;
    t.n0 = 0;
    t.nk = (25 * W::C1 + 63) / 64;
    t.n_mma = W::C2 < 16 ? 16 : W::C2;
  }
  __device__ void init_stage(const TcTile&, uint8_t*, uint8_t*) const {}
  __device__ uint32_t tx_bytes(const TcTile& t, int kb) const { return 16384 + 8 * 16 * W::C2; }
  __device__ void tma_issue(const TcTile& t, int kb, uint32_t a, uint32_t b, uint32_t mbar) const {
    const int r = t.m0 >> 8, y0 = (t.m0 >> 4) & 15;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = kb * 64 + 8 * j, tap = k >> W::L1, cc = k & (W::C1 - 1), ky = tap / 5, kx = tap - ky * 5;
      tc::tma_load_4d(a + 2048 * j, tmap_of(t, TM_A1), mbar, cc, kx - 2, tap < 25 ? y0 + ky - 2 : -64, r);
      tc::tma_load_2d(b + 16 * W::C2 * j, tmap_of(t, TM_W2F), mbar, k, 0);
    }
  }
  __device__ uint64_t a_desc(const TcTile&, uint32_t base, int ks) const {
    return tc::sdesc(base + 4096 * ks, 2048, 128);
  }
  __device__ uint64_t b_desc(const TcTile&, uint32_t base, int ks) const {
    return tc::sdesc(base + 32 * W::C2 * ks, 16 * W::C2, 128);
  }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
    // natural pixel order: a warp holds image rows y (lanes 0-15) and y+1 (lanes 16-31)
    constexpr int N = W::C2 < 16 ? W::C2 : 16;
    const int lane = threadIdx.x & 31, base = lane & 14;
    const int m = t.m0 + row, r = m >> 8, y = (m >> 4) & 15, x = m & 15;
    float val[16], best[16];
    int arg[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) val[j] = j < N ? fmaxf(v[j] + t.c->params[d.b2 + c0 + j], 0.f) : 0.f;
    pool_lanes(val, base, base + 1, base + 16, base + 17, best, arg);
    if (lane < 16 && (lane & 1) == 0) {
      const int64_t o = ((int64_t)r * 64 + (y >> 1) * 8 + (x >> 1)) * W::C2 + c0;
      st_bf16<N>((bf16*)t.c->buf[B_A2] + o, best);
      st_u8<N>((uint8_t*)t.c->buf[B_I2] + o, arg);
    }
  }
};

template <int WQ>
struct TmaConv2Wgrad : TcConv2Wgrad<WQ> {  // split-K over 2048-pixel chunks -> partial[split][C2][25 C1 + 1]
  typedef CnnW<WQ> W;
  static constexpr bool TMA = true;
  static constexpr int MT = (25 * W::C1 + 1 + 127) / 128;  // M tiles
  __device__ void setup(TcTile& t, int local) const {
    const int split = local / MT;
    t.m0 = (local - split * MT) * 128;
    t.n0 = split;
    const int kbs = t.tk.rows * 4 - split * (kWgradChunkPx / 64);
    t.nk = kbs < kWgradChunkPx / 64 ? kbs : kWgradChunkPx / 64;
    t.n_mma = W::C2 < 16 ? 16 : W::C2;
  }
  __device__ void init_stage(const TcTile& t, uint8_t* a, uint8_t* b) const {
    // m groups at/after the bias row: constant chunks ([1,0..] per pixel, or zeros), 64 rows x 16 B each
    for (int g = 0; g < 16; ++g) {
      const int mg = t.m0 + 8 * g, Kw = 25 * W::C1;
      if (mg < Kw) continue;
      const uint4 val = mg == Kw ? make_uint4(0x3F80u, 0, 0, 0) : make_uint4(0, 0, 0, 0);
      for (int i = threadIdx.x; i < 64; i += kTcProd) reinterpret_cast<uint4*>(a + 1024 * g)[i] = val;
    }
  }
  __device__ uint32_t tx_bytes(const TcTile& t, int kb) const {
    const int valid = (25 * W::C1 - t.m0) / 8;  // m groups loaded by TMA
    return 1024u * (valid < 16 ? (valid < 0 ? 0 : valid) : 16) + 1024u * (W::C2 / 8);
  }
  __device__ void tma_issue(const TcTile& t, int kb, uint32_t a, uint32_t b, uint32_t mbar) const {
    const int kg = t.n0 * (kWgradChunkPx / 64) + kb, r = kg >> 2, y0 = (kg & 3) * 4;
    for (int g = 0; g < 16; ++g) {
      const int mg = t.m0 + 8 * g;
      if (mg >= 25 * W::C1) break;
      const int tap = mg >> W::L1, cc = mg & (W::C1 - 1), ky = tap / 5, kx = tap - ky * 5;
      tc::tma_load_4d(a + 1024 * g, tmap_of(t, TM_A1W), mbar, cc, kx - 2, y0 + ky - 2, r);
    }
#pragma unroll
    for (int nc = 0; nc < W::C2 / 8; ++nc) tc::tma_load_4d(b + 1024 * nc, tmap_of(t, TM_DZ2W), mbar, 8 * nc, 0, y0, r);
  }
  __device__ uint64_t a_desc(const TcTile&, uint32_t base, int ks) const { return tc::sdesc(base + 256 * ks, 128, 1024); }
  __device__ uint64_t b_desc(const TcTile&, uint32_t base, int ks) const { return tc::sdesc(base + 256 * ks, 128, 1024); }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
    const int m = t.m0 + row, N = 25 * W::C1 + 1;
    if (m >= N) return;
    float* part = (float*)t.c->buf[B_WSP] + (int64_t)t.n0 * W::C2 * N + m;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (c0 + j < W::C2) part[(int64_t)(c0 + j) * N] = v[j];
  }
  // The last split of each (client, M tile) to finish sums the partials in split order (deterministic) and
  // applies the SGD update to the fp32 master and the bf16 shadow (fused reduce).  Counters: stats[8 + mtile].
  static constexpr bool FINISH = true;
  __device__ void finish(const TcTile& t) const {
    __shared__ int last;
    int* cnt = reinterpret_cast<int*>(t.c->stats) + 8 + t.m0 / 128;
    const int splits = (t.tk.rows * 256 + kWgradChunkPx - 1) / kWgradChunkPx;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(cnt, 1) == splits - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int N = 25 * W::C1 + 1, Kw = 25 * W::C1;
    const float* part = (const float*)t.c->buf[B_WSP];
    float* P = t.c->params;
    bf16* S = (bf16*)t.c->buf[B_WSH];
    for (int e = threadIdx.x; e < 128 * W::C2; e += blockDim.x) {
      const int m = t.m0 + (e & 127), co = e >> 7;
      if (m >= N) continue;
      float g = 0.f;
      for (int sp = 0; sp < splits; ++sp) g += __ldcg(part + ((int64_t)sp * W::C2 + co) * N + m);
      if (m < Kw) {
        const int64_t idx = this->d.w2 + (int64_t)co * Kw + m;
        const float nw = P[idx] - this->lr * g;
        P[idx] = nw;
        S[idx] = __float2bfloat16_rn(nw);
      } else {
        P[this->d.b2 + co] -= this->lr * g;
      }
    }
    if (threadIdx.x == 0) *cnt = 0;
  }
};

__device__ __forceinline__ int batch_rows16(const TcTile& t) { return (t.c->B + 15) & ~15; }

// fc1 operands are wide (K1 = 64 C2, F = 128 w): 64-element (128 B) TMA boxes with
// 128-byte swizzle, one box per operand (or two for the MN-major W^T) per K block.
template <int WQ>
struct TmaFc1Fwd : TcFc1Fwd<WQ> {
  typedef CnnW<WQ> W;
  static constexpr bool TMA = true;
  __device__ void init_stage(const TcTile&, uint8_t*, uint8_t*) const {}
  __device__ uint32_t tx_bytes(const TcTile& t, int kb) const { return 16384 + 128 * batch_rows16(t); }
  __device__ void tma_issue(const TcTile& t, int kb, uint32_t a, uint32_t b, uint32_t mbar) const {
    tc::tma_load_3d(a, tmap_of(t, TM_W3K), mbar, (kb & 1) * 64, kb >> 1, t.m0);  // [128 f][64 k] swizzled
    tc::tma_load_2d(b, tmap_of(t, TM_A2), mbar, kb * 64, 0);      // [R rows][64 k] swizzled
  }
  __device__ uint64_t a_desc(const TcTile&, uint32_t base, int ks) const {
    return tc::sdesc_sw128(base + 32 * ks, 16, 1024);
  }
  __device__ uint64_t b_desc(const TcTile& t, uint32_t base, int ks) const {
    return tc::sdesc_sw128(base + 32 * ks, 16, 1024);
  }
};

template <int WQ>
struct TmaFc1Dgrad : TcFc1Dgrad<WQ> {
  typedef CnnW<WQ> W;
  static constexpr bool TMA = true;
  __device__ void init_stage(const TcTile&, uint8_t*, uint8_t*) const {}
  __device__ uint32_t tx_bytes(const TcTile& t, int kb) const { return 16384 + 128 * batch_rows16(t); }
  __device__ void tma_issue(const TcTile& t, int kb, uint32_t a, uint32_t b, uint32_t mbar) const {
    tc::tma_load_3d(a, tmap_of(t, TM_W3M), mbar, 0, t.m0 >> 7, kb * 64);          // [64 f][64 m] swizzled
    tc::tma_load_3d(a + 8192, tmap_of(t, TM_W3M), mbar, 64, t.m0 >> 7, kb * 64);  // next 64 m
    tc::tma_load_2d(b, tmap_of(t, TM_DH), mbar, kb * 64, 0);                 // [R rows][64 f] swizzled
  }
  __device__ uint64_t a_desc(const TcTile&, uint32_t base, int ks) const {
    return tc::sdesc_sw128(base + 2048 * ks, 8192, 1024);  // MN-major: 16 k rows per step, 64-m blocks 8 KB apart
  }
  __device__ uint64_t b_desc(const TcTile& t, uint32_t base, int ks) const {
    return tc::sdesc_sw128(base + 32 * ks, 16, 1024);
  }
};

template <int WQ>
struct TmaFc1Wgrad : TcFc1Wgrad<WQ> {
  // Operands by TMA (no cp.async: its 16-byte chunk writes into the MN-major operand layout measured up to
  // 28-way shared-memory bank conflicts, 43 % of the kernel's shared wavefronts): A = a2 [R rows][64 k1] x 2,
  // B = dh [R rows][64 f] x 2 (128-byte swizzle, MN-major: K = rows at 128 B, 8-row groups 1 KB apart, the
  // two 64-wide atoms 8 KB apart); R = the slot's rows rounded to 16 (rows past the slot are the TMA's zero
  // fill; rows of a ragged batch past tk.rows are zero in dh: k_head_cnn).  K steps = R / 16.
  static constexpr bool TMA = true, KSTEPS = true;
  __device__ int ksteps(const TcTile& t) const { return ((t.c->B + 15) & ~15) >> 4; }
  __device__ void init_stage(const TcTile&, uint8_t*, uint8_t*) const {}
  __device__ uint32_t tx_bytes(const TcTile& t, int) const { return 512u * (uint32_t)((t.c->B + 15) & ~15); }
  __device__ void tma_issue(const TcTile& t, int, uint32_t a, uint32_t b, uint32_t mbar) const {
    tc::tma_load_2d(a, tmap_of(t, TM_A2), mbar, t.m0, 0);
    tc::tma_load_2d(a + 8192, tmap_of(t, TM_A2), mbar, t.m0 + 64, 0);
    tc::tma_load_2d(b, tmap_of(t, TM_DH), mbar, t.n0, 0);
    tc::tma_load_2d(b + 8192, tmap_of(t, TM_DH), mbar, t.n0 + 64, 0);
  }
  __device__ uint64_t a_desc(const TcTile&, uint32_t base, int ks) const {
    return tc::sdesc_sw128(base + 2048 * ks, 8192, 1024);
  }
  __device__ uint64_t b_desc(const TcTile&, uint32_t base, int ks) const {
    return tc::sdesc_sw128(base + 2048 * ks, 8192, 1024);
  }
};

// --------------------------------------------------------------------------
// conv1 on tensor cores.  K1 (staging): the batch is staged as bf16 x/255 with a
// 2-pixel zero border and the 3 channels padded to 8 (one aligned 16-byte chunk
// per pixel), columns split by parity: xs[r][Y 36][X % 2][X / 2 (18)][8] for the
// padded coordinates (Y, X) = (y + 2, x + 2).  Channel 3 is 1.0 inside the image
// (0 in the border): the conv1 wgrad reads the bias gradient from it.
// --------------------------------------------------------------------------
constexpr int kStageThreads = 256, kStagePx = 4;
__global__ void __launch_bounds__(kStageThreads)
    k_stage_x(const ClientRec* __restrict__ recs, const Task* __restrict__ tasks) {  // grid (blocks, task)
  // kStagePx staged pixels per thread (e = block base + k * 256 + thread): the task / record / permutation
  // loads are paid once per thread and all pixel loads are in flight together
  __shared__ float lut[256];  // px01(u): the same fp32 values as the division, without one per channel
  lut[threadIdx.x] = px01((uint8_t)threadIdx.x);
  pdl_wait();  // xs is still read by the preceding conv1 wgrad
  pdl_trigger();
  const Task tk = tasks[blockIdx.y];
  const int n_e = tk.rows * 1296, e0 = blockIdx.x * kStageThreads * kStagePx + threadIdx.x;
  if ((int)blockIdx.x * kStageThreads * kStagePx >= n_e) return;
  const ClientRec* c = recs + tk.rec;
  const uint8_t* xbase = c->x;
  uint4* xs = reinterpret_cast<uint4*>(c->buf[B_XS]);
  uint32_t u[kStagePx][3];
  bool in[kStagePx];
#pragma unroll
  for (int k = 0; k < kStagePx; ++k) {
    const int e = e0 + k * kStageThreads;
    const int r = e / 1296, rem = e - r * 1296, Y = rem / 36, rx = rem - Y * 36, X = 2 * (rx % 18) + rx / 18;
    const int y = Y - 2, x = X - 2;
    in[k] = e < n_e && (unsigned)y < 32u && (unsigned)x < 32u;
    u[k][0] = u[k][1] = u[k][2] = 0;
    if (in[k]) {
      const uint8_t* px = xbase + (int64_t)__ldg(c->perm + tk.base + r) * 3072 + (y * 32 + x) * 3;
      u[k][0] = __ldg(px), u[k][1] = __ldg(px + 1), u[k][2] = __ldg(px + 2);
    }
  }
  __syncthreads();  // lut
#pragma unroll
  for (int k = 0; k < kStagePx; ++k) {
    const int e = e0 + k * kStageThreads;
    if (e >= n_e) break;
    uint4 out = make_uint4(0, 0, 0, 0);
    if (in[k]) {
      const __nv_bfloat162 v01 = __floats2bfloat162_rn(lut[u[k][0]], lut[u[k][1]]);
      const __nv_bfloat162 v23 = __floats2bfloat162_rn(lut[u[k][2]], 1.f);
      out.x = *reinterpret_cast<const uint32_t*>(&v01);
      out.y = *reinterpret_cast<const uint32_t*>(&v23);
    }
    xs[e] = out;
  }
}
__device__ __forceinline__ int64_t xs_index(int r, int Y, int X) {  // 8-element chunk index of padded (Y, X)
  return ((int64_t)(r * 36 + Y) * 2 + (X & 1)) * 18 + (X >> 1);
}

// conv1 wgrad: D[m = tap*8 + ci (+ bias row 200), n = co] = sum_p xs(p, tap, ci) dz1[p][co],
// split-K over 2048-pixel chunks; the epilogue stores the 75 real rows + bias as
// partial[split][76][C1] (fp32), summed in split order by k_reduce_conv1_tc.
template <int WQ>
struct TcConv1Wgrad {
  typedef CnnW<WQ> W;
  static constexpr bool A_MN = true, B_MN = true;
  struct PA { int i, ky, kx, kind; };  // kind 0: gather tap (ky, kx), 1: ones, 2: zero
  struct PB { int i, n0; };
  const ClientRec* recs;
  CnnDims d;
  __device__ void setup(TcTile& t, int local) const {
    const int split = local >> 1;
    t.m0 = (local & 1) * 128;
    t.n0 = split;  // carries the split index
    const int px = t.tk.rows * 1024 - split * kWgradChunkPx;
    t.nk = (px < kWgradChunkPx ? px : kWgradChunkPx) / 64;
    t.n_mma = W::C1 < 16 ? 16 : W::C1;
  }
  __device__ const void* any(const TcTile& t) const { return t.c->params; }
  __device__ PA a_pre(const TcTile& t, int i, int j) const {
    const int tap = (t.m0 >> 3) + j;
    if (tap == 25) return PA{i, 0, 0, 1};
    if (tap > 25) return PA{i, 0, 0, 2};
    const int ky = tap / 5, kx = tap - ky * 5;
    return PA{i, ky, kx, 0};
  }
  __device__ const void* a_src(const TcTile& t, const PA& s, int kb) const {
    if (s.kind) return s.kind == 1 ? (const void*)kOneChunk : nullptr;
    const int p = t.n0 * kWgradChunkPx + kb * 64 + s.i, r = p >> 10, y = (p >> 5) & 31, x = p & 31;
    return (const bf16*)t.c->buf[B_XS] + xs_index(r, y + s.ky, x + s.kx) * 8;
  }
  __device__ PB b_pre(const TcTile& t, int i, int j) const { return PB{i, 8 * j}; }
  __device__ const void* b_src(const TcTile& t, const PB& s, int kb) const {
    if (s.n0 >= W::C1) return nullptr;
    const int p = t.n0 * kWgradChunkPx + kb * 64 + s.i;
    return (const bf16*)t.c->buf[B_DZC1] + (int64_t)p * W::C1 + s.n0;
  }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
    const int m = t.m0 + row;
    int idx;
    if (m == 200)
      idx = 75;
    else if (m < 200 && (m & 7) < 3)
      idx = (m >> 3) * 3 + (m & 7);
    else
      return;
    float* part = (float*)t.c->buf[B_WSP] + ((int64_t)t.n0 * 76 + idx) * W::C1;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (c0 + j < W::C1) part[c0 + j] = v[j];
  }
};

// Sum the split partials of element e = idx * C1 + co (idx 0..74 = weight (tap, ci), 75 = bias) in split
// order and apply SGD to the fp32 master and the pool-quad bf16 shadow (common.h w1q_index).
__device__ __forceinline__ void conv1_reduce_update(const ClientRec* c, int splits, int C1, int64_t off_w,
                                                    int64_t off_b, float lr, int e, int pbuf = B_WSP) {
  const int total = 76 * C1;
  const float* part = (const float*)c->buf[pbuf];  // split partials [splits][76 C1]
  float g = 0.f;
  for (int s0 = 0; s0 < splits; s0 += 8) {  // 8 independent loads in flight, summed in split order
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = s0 + j < splits ? __ldcg(part + (int64_t)(s0 + j) * total + e) : 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (s0 + j < splits) g += v[j];
  }
  const int idx = e / C1, co = e - idx * C1;
  if (idx == 75) {
    c->params[off_b + co] -= lr * g;
  } else {
    float* w = c->params + off_w + co * 75 + idx;
    const float nw = *w - lr * g;
    *w = nw;
    const int tap = idx / 3, ky = tap / 5, kx = tap - ky * 5, ci = idx - 3 * tap;
    const bf16 h = __float2bfloat16_rn(nw);
#pragma unroll
    for (int q = 0; q < 4; ++q)  // the weight's 4 places in the pool-quad shadow
      ((bf16*)c->buf[B_W1P])[w1q_index(C1, ky + (q >> 1), kx + (q & 1), q, co, ci)] = h;
  }
}

__global__ void __launch_bounds__(kReduceBlock)
    k_reduce_conv1_tc(const ClientRec* __restrict__ recs, const Task* __restrict__ tasks, const int* __restrict__ prefix,
                      int ntask, int C1, int64_t off_w, int64_t off_b, float lr) {
  const int ti = find_task(prefix, ntask, blockIdx.x);
  const Task tk = tasks[ti];
  const ClientRec* c = recs + tk.rec;
  const int e = (blockIdx.x - __ldg(prefix + ti)) * kReduceBlock + threadIdx.x;
  if (e >= 76 * C1) return;
  conv1_reduce_update(c, cdiv(tk.rows * 1024, kWgradChunkPx), C1, off_w, off_b, lr, e);
}

// --------------------------------------------------------------------------
// self-test GEMM (protea_selftest_gemm): D[M,N] = A B^T with dense bf16 operands
// --------------------------------------------------------------------------
struct TcDense {  // A [M][K], B [N][K] (K-major)
  static constexpr bool A_MN = false, B_MN = false;
  struct PA { const bf16* p; };
  struct PB { const bf16* p; };
  const ClientRec* recs;
  const bf16* A;
  const bf16* B;
  float* D;
  int M, N, K;
  __device__ void setup(TcTile& t, int local) const {
    t.m0 = local * 128;
    t.n0 = 0;
    t.nk = K / 64;
    t.n_mma = round16(N);
  }
  __device__ const void* any(const TcTile& t) const { return A; }
  __device__ PA a_pre(const TcTile& t, int i, int j) const { return PA{A + (int64_t)(t.m0 + i) * K + 8 * j}; }
  __device__ const void* a_src(const TcTile& t, const PA& s, int kb) const { return s.p + kb * 64; }
  __device__ PB b_pre(const TcTile& t, int i, int j) const { return PB{i < N ? B + (int64_t)i * K + 8 * j : nullptr}; }
  __device__ const void* b_src(const TcTile& t, const PB& s, int kb) const { return s.p ? s.p + kb * 64 : nullptr; }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (c0 + j < N) D[(int64_t)(t.m0 + row) * N + c0 + j] = v[j];
  }
};

struct TcDenseMN {  // A given as [K][M] (MN-major), B as [K][N] (MN-major)
  static constexpr bool A_MN = true, B_MN = true;
  struct PA { const bf16* p; };
  struct PB { const bf16* p; };
  const ClientRec* recs;
  const bf16* A;
  const bf16* B;
  float* D;
  int M, N, K;
  __device__ void setup(TcTile& t, int local) const {
    t.m0 = local * 128;
    t.n0 = 0;
    t.nk = K / 64;
    t.n_mma = round16(N);
  }
  __device__ const void* any(const TcTile& t) const { return A; }
  __device__ PA a_pre(const TcTile& t, int i, int j) const { return PA{A + (int64_t)i * M + t.m0 + 8 * j}; }
  __device__ const void* a_src(const TcTile& t, const PA& s, int kb) const { return s.p + (int64_t)kb * 64 * M; }
  __device__ PB b_pre(const TcTile& t, int i, int j) const {
    return PB{8 * j < N ? B + (int64_t)i * N + 8 * j : nullptr};
  }
  __device__ const void* b_src(const TcTile& t, const PB& s, int kb) const {
    return s.p ? s.p + (int64_t)kb * 64 * N : nullptr;
  }
  __device__ void epilogue(const TcTile& t, int row, int c0, const float (&v)[16]) const {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (c0 + j < N) D[(int64_t)(t.m0 + row) * N + c0 + j] = v[j];
  }
};

}  // namespace protea
