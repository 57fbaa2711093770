/*
 * protea.h — C ABI of the B200-native Protea hot path.
 *
 * What the library does (PAPER.md = the Protea paper, arXiv 2207.01053):
 *   - profile clients: peak device bytes + device-timed training time
 *     (Table 1 "VRAM", "CUDA_time", §2.2; get_properties() P:217 §3.3);
 *   - plan: turn profiles into GPU memory slots and a FIFO admission schedule
 *     (Eq. (1) P:243-249 §3.4; VCE stages (1)-(4) P:209 §3.2);
 *   - run one federated round: every sampled client's local SGD epochs on its
 *     own shard with its own batch size / model width, then sample-weighted
 *     FedAvg (§3.3 configure_fit / aggregate_fit);
 *   - FedAvg of arbitrary device vectors (McMahan et al. P:83).
 *
 * Conventions (apply to every call):
 *   - Ownership: the caller owns every array it passes and must keep it alive
 *     for the duration of the call only.  The library never retains caller
 *     pointers, EXCEPT the arena block given to protea_init, which must outlive
 *     the context.  The library owns (and frees in protea_finalize) its device
 *     copies of shards and its workspace.
 *   - Errors: every call returns a protea_status.  Validation runs before any
 *     device work, so on error no output is written.  protea_last_error()
 *     returns a message naming the offending client / field.
 *   - Threading: one context per GPU / rank; a context is not thread-safe.
 *     protea_plan is a pure host function (no context) and deterministic, so
 *     every rank computes the identical plan.
 *   - Pointers: "device" = CUDA device memory of the context's GPU; "host" =
 *     ordinary (preferably pinned) host memory.  protea_run_round accepts
 *     either for global_in / global_out (cudaPointerGetAttributes decides).
 *   - Streams: all device work is ordered on the stream given at init; calls
 *     return after that stream is synchronised.
 */
#ifndef PROTEA_H
#define PROTEA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PROTEA_OK = 0,
  PROTEA_ERR_INVALID = 1,     /* null pointer, n == 0, batch/epochs <= 0, n_k <= 0, unknown model, duplicate id */
  PROTEA_ERR_EMPTY = 2,       /* no results to aggregate */
  PROTEA_ERR_ZERO_WEIGHT = 3, /* sum of num_examples == 0 */
  PROTEA_ERR_DIM = 4,         /* dimension mismatch */
  PROTEA_ERR_NO_CAPACITY = 5, /* a slot exceeds every GPU's capacity (rejected, not clamped) */
  PROTEA_ERR_PLAN = 6,        /* plan/client mismatch, overlap, slot too small, missing client */
  PROTEA_ERR_OOM = 7,         /* arena overrun: the plan does not fit the arena */
  PROTEA_ERR_CUDA = 8,
  PROTEA_ERR_NCCL = 9
} protea_status;

enum { PROTEA_MODEL_MLP = 0, PROTEA_MODEL_CNN = 1, PROTEA_MODEL_RESNET8 = 2, PROTEA_MODEL_RESNET18 = 3 };
enum { PROTEA_PREC_FP32 = 0, PROTEA_PREC_BF16 = 1 };
enum { PROTEA_POLICY_PROFILED = 0, PROTEA_POLICY_STATIC = 1 };
enum { PROTEA_ORDER_ASC_ID = 0, PROTEA_ORDER_DESC_STEPS = 1 };

typedef struct protea_ctx protea_ctx;

typedef struct {
  int32_t device;          /* CUDA device ordinal of this rank */
  int32_t rank;            /* this rank in [0, world) */
  int32_t world;           /* number of ranks (GPUs); 1 = no NCCL */
  int32_t precision;       /* PROTEA_PREC_*: activation storage + GEMM operand type */
  const uint8_t* nccl_id;  /* host, 128 bytes (ncclUniqueId from rank 0, broadcast by the caller); NULL: no NCCL
                              communicator (world == 1, or caller-side reduction via partial_only rounds).
                              Given (also with world == 1), protea_run_round agrees on the plan and on every
                              rank's validation verdict through the communicator before any device work, and
                              exchanges the FedAvg partials with ncclAllGather + a rank-ordered sum (K7) */
  void* arena;             /* device, caller-owned block holding the client slots (e.g. a torch uint8 tensor) */
  uint64_t arena_bytes;    /* capacity C_g of this GPU's arena */
  void* stream;            /* cudaStream_t to order all work on (NULL = the legacy default stream) */
} protea_init_opts;

/* Model family of a shape group.  CNN: width = width_q / 4, width_q in {1,2,4}
 * (BASELINE.json configs[3]); MLP / RESNET8 / RESNET18 require width_q == 4.
 * H, W, C: input image shape (MLP 28x28x1; CNN 32x32x3 CIFAR-shaped, or 28x28x1 FEMNIST-shaped, the paper's
 * LEAF experiment P:304; RESNET8 / RESNET18 32x32x3).  RESNET18 is the paper's CIFAR model with
 * GroupNorm (2 groups) after every conv and option-A shortcuts (reading R26); it runs on the SIMT
 * kernels in both precisions. */
typedef struct {
  int32_t arch;      /* PROTEA_MODEL_* */
  int32_t width_q;
  int32_t classes;
  int32_t H, W, C;
} protea_model_desc;

/* One client's data shard: n_k examples, NHWC u8 pixels x[n*H*W*C], labels y[n] in [0, classes). Host pointers. */
typedef struct {
  int64_t client_id;
  int64_t n;
  const uint8_t* x;
  const int32_t* y;
} protea_shard;

/* One sampled client of a round. */
typedef struct {
  int64_t client_id;
  int32_t model_id;  /* from protea_register_model */
  int32_t batch;     /* B_k > 0 */
  int32_t epochs;    /* E > 0 */
  int32_t reserved;
} protea_client;

/* get_properties() record; integer SI units. */
typedef struct {
  int64_t client_id;
  uint64_t peak_bytes;  /* arena high-water mark of the client's slot (Table 1 VRAM): protea_profile_clients and
                           observe_hwm rounds report the OBSERVED mark (poisoned slot, highest touched byte,
                           aligned to 256 B); otherwise the slot layout's bound */
  uint64_t steps;       /* S_k = E * ceil(n_k / B_k) */
  uint64_t flops;       /* E * n_k * f(model, width) */
  uint64_t step_ns;     /* device time of one local step: in protea_profile_clients the marginal cost of a
                           step, median two-step run - median one-step run of the client alone (CUDA events;
                           admission and table upload cancel; >= 1000); train_ns / steps in the in-run
                           profiles of protea_run_round */
  uint64_t train_ns;    /* probe: step_ns * steps; in-run: sm_ns / #SMs (the client's SM-time share as
                           whole-GPU time) — Table 1 CUDA_time */
  uint64_t sm_ns;       /* in-run: sum of the durations of the CTAs that worked for the client (globaltimer;
                           persistent kernels split a CTA's time by tile count); 0 in probe profiles */
  uint32_t uses_gpu;    /* 1 */
  uint32_t reserved;
} protea_profile;

typedef struct {
  uint32_t n_gpus;            /* G >= 1 */
  uint32_t reserved;
  const uint64_t* capacity;   /* host, C_g for g in [0, G) (bytes) */
} protea_cluster;

typedef struct {
  int32_t policy;             /* PROTEA_POLICY_PROFILED (slots from profiles) or _STATIC (one client per GPU) */
  int32_t order;              /* PROTEA_ORDER_ASC_ID (paper FIFO) or _DESC_STEPS */
  uint32_t margin_permille;   /* slot = align256(ceil(peak * margin / 1000)); >= 1000 */
  uint32_t max_active;        /* 0 = unlimited */
} protea_plan_opts;

typedef struct {
  int64_t client_id;
  int32_t gpu;
  uint32_t q1024;    /* Eq. (1): ceil(1024 * slot / sum_g C_g) — num_gpus in units of 1/1024 */
  uint64_t offset;   /* slot offset in the GPU's arena */
  uint64_t slot;     /* slot bytes */
  uint64_t admit;    /* first lock-step iteration */
  uint64_t release;  /* admit + S_k */
} protea_assignment;

/* Op classes of one lock-step iteration (kernel families), for per-op timing
 * and the algorithmic work counters of protea_round_stats. */
enum {
  PROTEA_OPC_CONV1_FWD = 0, PROTEA_OPC_CONV2_FWD, PROTEA_OPC_FC1_FWD, PROTEA_OPC_HEAD, PROTEA_OPC_FC1_DGRAD,
  PROTEA_OPC_FC1_WGRAD, PROTEA_OPC_CONV2_DGRAD, PROTEA_OPC_CONV2_WGRAD, PROTEA_OPC_CONV2_REDUCE,
  PROTEA_OPC_CONV1_WGRAD, PROTEA_OPC_CONV1_REDUCE, PROTEA_OPC_MLP_FC1_FWD, PROTEA_OPC_MLP_HEAD,
  PROTEA_OPC_MLP_FC1_WGRAD, PROTEA_OPC_ADMIT, PROTEA_OPC_FEDAVG, PROTEA_OPC_STAGE_X,
  PROTEA_OPC_R_FWD, PROTEA_OPC_R_HEAD, PROTEA_OPC_R_DGRAD, PROTEA_OPC_R_WGRAD, PROTEA_OPC_R_REDUCE, /* ResNet-8 */
  PROTEA_OPC_EVAL_HEAD, /* evaluate round: classifier head after the forward kernels */
  PROTEA_OPC_G_FWD, PROTEA_OPC_G_NORM, PROTEA_OPC_G_HEAD, PROTEA_OPC_G_DGRAD, PROTEA_OPC_G_WGRAD,
  PROTEA_OPC_G_REDUCE, /* ResNet-18 (GroupNorm): conv fwd, GroupNorm fwd / bwd, head, conv dgrad, wgrad, reduces */
  PROTEA_N_OPC = 32 /* room for further op classes */
};

typedef struct {
  float lr;          /* SGD learning rate eta */
  uint32_t seed;     /* permutation seed (oracle/splitmix reading R10) */
  uint32_t round;    /* round index */
  int32_t shuffle;   /* 1 = SplitMix64 epoch permutation, 0 = identity order */
  uint32_t time_ops; /* bitmask over PROTEA_OPC_*: bracket every launch of those classes with CUDA events */
  uint32_t partial_only; /* 1: skip the cross-rank sum and the finalisation; keep this rank's fp64 FedAvg
                            partial (protea_round_partial) for a caller-side reduction (protea_round_finalize);
                            global_out is not written */
  uint32_t serialize;    /* 1: every launch on the lock-step stream (no fc1-wgrad deferral to the side
                            stream), so per-op CUDA-event times are the kernels' own, as in a serialised
                            ncu launch list; 0: default overlap */
  uint32_t observe_hwm;  /* 1: OBSERVE each client's arena high-water mark (Table 1 VRAM): its slot
                            is filled with the poison byte PROTEA_POISON at admission and scanned at release;
                            measured[k].peak_bytes = align256(1 + offset of the highest byte of the slot that
                            differs from the poison).  0: measured[k].peak_bytes = the slot layout's bound */
  uint32_t n_trace;      /* verification: number of traced clients (0 = none) */
  const int64_t* trace_ids;   /* host, n_trace client ids (this rank's) */
  void* const* trace_bufs;    /* host array of n_trace DEVICE pointers, each (S_k + 1) * H_k bytes with H_k =
                                 protea_client_footprint's peak_bytes (the slot layout): snapshot s
                                 = the client's whole slot after s local steps (s = 0: at admission) — fp32
                                 weights first, then the step's stored activations / decisions (pool argmaxes) */
} protea_round_opts;

#define PROTEA_POISON 0xA5 /* byte value of an untouched slot byte under observe_hwm */

typedef struct {
  uint64_t round_ns;        /* device time of the whole round on this rank (CUDA events) */
  uint64_t iterations;      /* lock-step iterations run on this rank (= makespan of its GPU) */
  uint64_t client_steps;    /* sum S_k over this rank's clients */
  uint64_t kernel_launches; /* kernels launched by the round on this rank */
  uint64_t flops;           /* sum FLOPs_k over this rank's clients */
  double loss_sum;          /* sum over this rank's client steps of the mean batch loss */
  uint64_t op_ns[PROTEA_N_OPC];       /* summed device time of the op classes selected by time_ops */
  uint64_t op_launches[PROTEA_N_OPC]; /* kernel launches per op class */
  uint64_t op_flops[PROTEA_N_OPC];    /* algorithmic FLOPs per op class (2 x useful MACs) */
  uint64_t op_bytes[PROTEA_N_OPC];    /* algorithmic (compulsory) HBM bytes per op class: operands read once, results written once */
  /* The launches behind op_ns and their algorithmic work.  Launches deferred to the low-priority side
   * stream (fc1 wgrad in light iterations, run concurrently with other kernels) are not timed. */
  uint64_t op_timed_launches[PROTEA_N_OPC];
  uint64_t op_timed_flops[PROTEA_N_OPC];
  uint64_t op_timed_bytes[PROTEA_N_OPC];
} protea_round_stats;

/* Create a context on opts->device: the simulation engine of one GPU (P:209 the VCE's per-GPU resource
 * pool, here the caller-owned arena of capacity C_g = opts->arena_bytes that client slots are packed into,
 * Eq. (1)).  world > 1 bootstraps an NCCL communicator from opts->nccl_id (multi-GPU placement,
 * P:334).  Errors: INVALID (bad field), CUDA, NCCL. */
protea_status protea_init(const protea_init_opts* opts, protea_ctx** out);

/* Free the context, its device copies and workspace (not the caller's arena). */
void protea_finalize(protea_ctx* ctx);

/* Message of the last failed call on ctx (or of the last failed context-free call when ctx == NULL). */
const char* protea_last_error(const protea_ctx* ctx);

/* Register a shape group (a model of P:304: MLP, CNN-w, ResNet-8 / ResNet-18, reading R11 / R26 / R27;
 * the groups of HeteroFL-style widths are FedAvg'd independently, reading R12).  Its global weights occupy
 * [offset, offset + n_params) of the concatenated global vector, groups in registration order; *n_params
 * receives P of this group.  All groups of a context take one input size (INVALID otherwise).
 * Errors: INVALID. */
protea_status protea_register_model(protea_ctx* ctx, const protea_model_desc* desc, int32_t* model_id,
                                    uint64_t* n_params);

/* Copy n shards to device (library-owned): each client's local data set (P:302 the per-client partitions;
 * synthetic here).  Re-registering an id replaces it.  Labels are range-checked against the
 * client's model when a round or profile uses the shard (INVALID there).
 * Errors: INVALID (null, n_k <= 0), CUDA. */
protea_status protea_register_shards(protea_ctx* ctx, const protea_shard* shards, size_t n);

/* Profile n clients (shards must be registered): peak bytes, S_k, FLOPs, and the device time of one probe
 * step per shape class (model, batch) run in the arena (which must not be in use).  peak_bytes is OBSERVED:
 * every client runs one local step (its epoch permutations for all E epochs, one batch) in a poisoned slot
 * of the layout's size followed by a 4 KiB poisoned guard; the highest touched byte of the slot, aligned to
 * 256 B, is the client's high-water mark, and a touched guard byte (a slot overrun) is an error.
 * out: caller-allocated, n records.
 * Errors: INVALID, OOM (arena smaller than a probe slot, or a guard byte touched), CUDA. */
protea_status protea_profile_clients(protea_ctx* ctx, const protea_client* clients, size_t n,
                                     protea_profile* out);

/* Pure host planner (no context): LPT partition by FLOPs across GPUs, then
 * per-GPU strict-FIFO admission replay with address first-fit.
 * out: caller-allocated n records, written in ascending client_id order;
 * makespan_steps: caller-allocated G entries.
 * Errors: INVALID, NO_CAPACITY, PLAN. */
protea_status protea_plan(const protea_profile* profiles, size_t n, const protea_cluster* cluster,
                          const protea_plan_opts* opts, protea_assignment* out, uint64_t* makespan_steps);

/* Result of evaluating a model on a set of samples (§4.1: every client
 * keeps a validation split; the evaluate round follows aggregation). */
typedef struct {
  double loss_sum;   /* sum over samples of the cross-entropy of the model's logits (fp32 forward, fp64 sum) */
  uint64_t correct;  /* samples whose first-maximum logit is the label */
  uint64_t n;        /* samples evaluated */
} protea_eval_result;

/* Evaluate registered model `model_id` (MLP or CNN-w) with `weights` (its n_params floats, host or device)
 * on n samples: x u8 [n][H][W][C] NHWC and y int32 [n], both host, copied by the library.  The forward
 * pass runs in fp32 on the verify-mode kernels over groups of 64 samples (one grouped launch per layer).
 * loss_sum / n is the mean validation loss, correct / n the accuracy.  Errors: INVALID (unknown or
 * ResNet model, n <= 0, null pointer, label outside [0, classes)), CUDA. */
protea_status protea_evaluate(protea_ctx* ctx, int32_t model_id, const float* weights, const uint8_t* x,
                              const int32_t* y, int64_t n, protea_eval_result* out);

/* Register clients' VALIDATION splits (§4.1: each client's data is split into training and
 * validation sets), same record and ownership as protea_register_shards, kept apart from the training
 * shards (re-registering an id replaces it).  Errors: INVALID (null, n_k <= 0, no model registered), CUDA. */
protea_status protea_register_val_shards(protea_ctx* ctx, const protea_shard* shards, size_t n);

/* Evaluate round (the server's configure_evaluate / aggregate_evaluate after aggregation; P:302 the
 * validation split): every listed client evaluates its group's global weights (n_params floats, all
 * groups concatenated, host or device) on its registered validation split.  The forward pass is the
 * training path's (bf16 mode: the tcgen05 kernels of every model; fp32 mode: the SIMT verify kernels), in
 * lock-step over all clients (batches above 64 rows as micro-clients), followed by a classifier head
 * (fp32 logits, logsumexp - z[y], first-maximum argmax).  per_client (caller-allocated, n records, in the
 * given order): loss_sum (sum of the per-sample cross-entropies), correct, n; total (nullable): their sums
 * (aggregate_evaluate: loss_sum / n is the example-weighted mean loss, correct / n the accuracy).  The
 * arena is used as scratch (must not be in use).  Errors: INVALID (null, unknown model, duplicate id, no
 * validation split, label outside [0, classes)), DIM, OOM (a client's evaluation slot exceeds the arena),
 * CUDA. */
protea_status protea_evaluate_round(protea_ctx* ctx, const protea_client* clients, size_t n, const float* global,
                                    size_t n_params, protea_eval_result* per_client, protea_eval_result* total);

/* 64-bit FNV-1a hash of a round's client list and plan (every field of both arrays, in the given
 * order).  Pure host function.  protea_run_round with world > 1 compares it across ranks before
 * any device work (NCCL max of h and ~h, SURVEY §8(e) "plan agreement"); ranks that were given
 * different plans or client lists fail with PROTEA_ERR_PLAN. */
uint64_t protea_plan_hash(const protea_client* clients, size_t n, const protea_assignment* plan);

/* Run one round.  Every rank passes the same clients and plan; this rank runs
 * the clients whose gpu == rank in lock-step iterations at their planned arena
 * offsets, then all ranks sum the per-GPU FedAvg partials (NCCL when world > 1)
 * and every rank writes the new global weights.
 * global_in / global_out: n_params floats (all registered groups concatenated),
 * host or device; a group without sampled clients is copied unchanged.
 * measured (nullable): n records of in-run profiles; stats (nullable).
 * With a communicator: the ranks' protea_plan_hash values must agree and every rank must pass its own
 * validation (else PLAN on the ranks that passed, nothing run anywhere); a rank failing during the round
 * is reported to all ranks before the exchange (CUDA).
 * Errors: INVALID, PLAN, OOM, CUDA, NCCL. */
protea_status protea_run_round(protea_ctx* ctx, const protea_round_opts* opts, const protea_client* clients,
                               size_t n, const protea_assignment* plan, const float* global_in, float* global_out,
                               size_t n_params, protea_profile* measured, protea_round_stats* stats);

/* Copy the fp64 FedAvg partial of the last protea_run_round (partial_only = 1) of
 * this rank: acc[d] = sum over this rank's clients of n_k (w_k[d] - w_g[d]),
 * n_params doubles, all groups concatenated.  dst: host or device.
 * Errors: INVALID (no partial round recorded, size mismatch), CUDA. */
protea_status protea_round_partial(protea_ctx* ctx, double* dst, size_t n_params);

/* Finish a partial round (= protea_round_finalize_ordered with one part): global_out = global_in +
 * acc_sum / N_group per shape group (N_group = sum n_k over ALL ranks' clients of that group, recorded by
 * the last protea_run_round; groups without clients are copied unchanged).
 * acc_sum: the element-wise sum of every rank's partial (device or host).
 * Errors: INVALID, DIM, CUDA. */
protea_status protea_round_finalize(protea_ctx* ctx, const double* acc_sum, const float* global_in, float* global_out,
                                    size_t n_params);

/* Deterministic cross-rank finalise (K7, SURVEY §8(e) "gather the partials, reduce in rank order"):
 * global_out = global_in + (((p_0 + p_1) + p_2) + ... + p_{nparts-1}) / N_group per shape group, the sum
 * in fp64 in rank order, one rounding to fp32 (reading R20).  partials: nparts consecutive
 * rank partials of n_params doubles each (protea_round_partial of ranks 0..nparts-1; device or host).
 * This is the kernel protea_run_round runs after its ncclAllGather when it holds a communicator, so the
 * multi-rank result equals this call on the same partials bit for bit.  N_group as in
 * protea_round_finalize.  Errors: INVALID (null, nparts < 1, no round recorded), DIM, CUDA. */
protea_status protea_round_finalize_ordered(protea_ctx* ctx, const double* partials, int32_t nparts,
                                            const float* global_in, float* global_out, size_t n_params);

/* HeteroFL-style overlapping-width aggregation for the CNN-w family (DESIGN.md
 * reading R23; the paper's FedAvg P:234 generalised to nested sub-models).  The global model is the
 * full-width CNN (width_q 4, `classes` outputs); a width-q client holds the sub-model of the first
 * C1 = 8q / C2 = 16q / F = 128q channels of every hidden dimension (fc1 inputs: the first C2 channels
 * of each of the 8x8 pooled positions; fc2: every class).
 * protea_heterofl_extract: sub_out (device, n_params(CNN, width_q) floats) = that sub-model of
 *   global_full (device, n_params(CNN, 4) floats).
 * protea_heterofl_aggregate: out[i] (device, full width) = the num_examples-weighted mean of element i
 *   over the clients whose sub-model holds it (fp64, in the given client order, one rounding), or
 *   global_full[i] when none does.  params: host array of n device pointers (client k: its width_q[k]
 *   sub-model); width_q, num_examples: host arrays of n.
 * Errors: INVALID (null, classes not in [2, 64], width not in {1, 2, 4}, n_k <= 0), EMPTY (n == 0),
 * CUDA.  Validation precedes device work. */
protea_status protea_heterofl_extract(protea_ctx* ctx, int32_t classes, const float* global_full, int32_t width_q,
                                      float* sub_out);
protea_status protea_heterofl_aggregate(protea_ctx* ctx, int32_t classes, const float* global_full,
                                        const float* const* params, const int32_t* width_q,
                                        const int64_t* num_examples, size_t n, float* out);

/* out[d] = sum_k n_k params[k][d] / sum_k n_k, fp64 accumulation in the given
 * order, one rounding to fp32.  params: host array of n device pointers, each
 * dim floats; out: device, dim floats.
 * Errors: EMPTY (n == 0), INVALID (null, n_k <= 0), ZERO_WEIGHT, CUDA. */
protea_status protea_fedavg(protea_ctx* ctx, const float* const* params, const int64_t* num_examples, size_t n,
                            size_t dim, float* out);

/* Host helpers (pure, no context) mirroring the profiler formulas, so callers
 * can plan without a GPU: slot bytes (exact HWM) and FLOPs of one client. */
protea_status protea_client_footprint(const protea_model_desc* desc, int64_t n, int32_t batch, int32_t epochs,
                                      int32_t precision, uint64_t* peak_bytes, uint64_t* steps, uint64_t* flops);

#ifdef __cplusplus
}
#endif
#endif /* PROTEA_H */
