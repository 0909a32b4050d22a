/*
 * fl.h — C-ABI of the B200-native FedAvg-round engine (Pollen, arXiv 2306.17453).
 *
 * One simulated FedAvg round (§2.1): the server sends θ_g to
 * every cohort client, each client runs E epochs of minibatch SGD on its own
 * ragged dataset, and the server forms the sample-count-weighted mean
 * (Eq. 1-2).  Around it: Pollen's push-based placement of the whole
 * cohort onto workers in one step (§4.1, §5), here one
 * worker = one GPU = one process (rank).
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; readings Ax =
 * DESIGN.md §"Readings of the paper".
 *
 * Conventions (all entry points):
 *  - Every function returns fl_status; no exception or abort crosses the ABI.
 *  - Host pointers are borrowed for the duration of the call unless stated.
 *  - Device pointers must be on cfg.device; borrowed, never freed by the library.
 *  - Outputs are caller-allocated.
 *  - Validation errors return FL_ERR_INVALID and leave the context unchanged.
 *  - A CUDA/NCCL failure latches the context into a FAILED state; every later
 *    call on it returns FL_ERR_STATE.  fl_last_error() describes the cause.
 *  - Determinism: the same inputs give bit-identical plans and segment
 *    offsets on every rank and every run; aggregation is deterministic for a
 *    fixed world size (fixed client order, fp64 accumulation).
 *  - There is no CPU fallback: entry points that compute need a CUDA device
 *    (sm_100a) and return FL_ERR_CUDA without one.  Only fl_place_plan,
 *    fl_pack_plan, fl_lb_fit, fl_n_params and fl_abi_version are host-only.
 */
#ifndef FL_B200_H
#define FL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FL_ABI_VERSION 3u

typedef enum {
  FL_OK = 0,
  FL_ERR_INVALID = 1,     /* bad argument; ctx unchanged */
  FL_ERR_STATE = 2,       /* call out of order, or ctx FAILED */
  FL_ERR_OOM = 3,         /* device allocation failed */
  FL_ERR_CUDA = 4,        /* CUDA runtime/launch error (or no device) */
  FL_ERR_NCCL = 5,        /* NCCL missing or failed */
  FL_ERR_EMPTY = 6,       /* total sample count is 0 */
  FL_ERR_UNSUPPORTED = 7  /* model/option not built in this version */
} fl_status;

typedef enum {
  FL_MODEL_LOGREG = 0,     /* 784 -> 10 softmax regression (BASELINE configs[0]) */
  FL_MODEL_CNN_CIFAR = 1,  /* McMahan CNN, 3x32x32, 'same' padding (reading A10) */
  FL_MODEL_CNN_SPEECH = 2, /* conv+MLP on 1x40x98 (reading A10) */
  FL_MODEL_CHAR_LSTM = 3   /* LEAF char-LSTM, embed 8, 2x256, seq 80 */
} fl_model;

/* Placement policies, §5 L358-388.  Clients are ordered by batch
 * count m = ceil(n/B) descending, ties by client id ascending (reading A15);
 * BU/LB append each client to the worker with the lowest load, ties to the
 * lowest worker id.  BU load = Σ m (L370); LB load = Σ Eq. 3
 * prediction a·m + b·ln(c·m) + d, clamped to >= 1e-12 (L380-388).
 * FL_PLACE_LB_GPU is LB with one Eq. 3 fit per GPU (lb_coef = [world_size][4]):
 * workers are ordered fastest-first by the predicted time of the cohort's largest
 * client (L385-386), each client goes to the worker with the lowest predicted load
 * Σ Eq. 3(coef[w], m), ties to the earlier worker in that order. */
typedef enum { FL_PLACE_BU = 0, FL_PLACE_LB = 1, FL_PLACE_RR = 2, FL_PLACE_SRR = 3,
               FL_PLACE_LB_GPU = 4 } fl_policy;

typedef struct fl_ctx fl_ctx; /* opaque; owns device buffers, stream, events, NCCL comm */

typedef struct {
  uint32_t abi_version;     /* must be FL_ABI_VERSION */
  int32_t model;            /* fl_model */
  int32_t batch_size;       /* B >= 1 */
  int32_t local_epochs;     /* E >= 1 */
  float lr;                 /* η >= 0: plain SGD, no momentum / decay (reading A8) */
  int32_t shuffle;          /* 0: stored order; 1: SplitMix64 Fisher-Yates per (seed, round, id, epoch) (A5) */
  uint64_t seed;
  int64_t min_samples;      /* clients with n < min_samples are rejected (P:447 exclusion, reading A6); >= 1 */
  int32_t rank, world_size; /* one process per GPU; 0 <= rank < world_size */
  int32_t device;           /* CUDA ordinal of this rank */
  const uint8_t* nccl_unique_id; /* 128 bytes from fl_nccl_unique_id() on rank 0; required if world_size > 1.
                                    With world_size == 1 a non-NULL id creates a 1-rank communicator and
                                    fl_aggregate takes the multi-rank path (partial [S‖N] -> ncclAllReduce ->
                                    finalize) on one GPU; NULL: the fused single-GPU accumulate+finalize. */
  int32_t math;             /* 0: tensor cores (TF32, tcgen05) where built; 1: FP32 SIMT everywhere */
  void* stream;             /* optional borrowed cudaStream_t; NULL: the ctx creates its own */
  /* SM partition of this rank (a CUDA green context; heterogeneous-worker emulation):
   *   0: the whole GPU;  s > 0: the first partition of >= s SMs of cfg.device;
   *   s < 0: the remainder after splitting off the first partition of >= -s SMs (so two ranks
   *   configured s and -s share a GPU on disjoint SMs).  Every stream of the ctx is created in
   *   the partition; persistent grids are sized to its SM count.  FL_ERR_INVALID with a
   *   borrowed stream; FL_ERR_CUDA if the driver cannot split. */
  int32_t sm_count;
  /* Cross-rank aggregation (world_size > 1), the paper's server-traffic question (P:73, P:221-222,
   * §4.3):
   *   FL_AGG_NCCL (0): per-GPU fused partial [S_g ‖ N_g] -> ncclAllReduce -> finalize;
   *   FL_AGG_PEER (1): one kernel per rank over peer memory: the fused fp64 partial S_g, then
   *     this rank's slice of Σ_g S_g read from every peer, θ_new = fp32(θ_g + S/N) stored into
   *     every rank's θ_g (reduce-scatter + finalize + all-gather, no NCCL); needs fl_peer_connect;
   *   FL_AGG_UNAGGREGATED (2): the ablation without partial aggregation: every rank ships each
   *     client model θ_k (fp32) to rank 0 (the "server GPU"), which averages all
   *     of them and stores θ_new into every rank; needs fl_peer_connect. */
  int32_t agg_mode;
} fl_config;

typedef enum { FL_AGG_NCCL = 0, FL_AGG_PEER = 1, FL_AGG_UNAGGREGATED = 2 } fl_agg_mode;

/* The client population, client-id order.  Sample rows of client k
 * are rows [Σ_{j<k} n_j, Σ_{j<=k} n_j) of x / y.
 *   logreg/CNN/speech: x = float32[rows][feature_dim] (CNN: C,H,W order), y = int32 class
 *   LSTM:              x = uint8[rows][80] characters, y = int32 next character
 * on_device = 1: x, y are device pointers on cfg.device, borrowed for the ctx lifetime.
 * on_device = 0: x, y are host pointers, borrowed for the ctx lifetime; each
 *   round copies this rank's cohort rows host->device (the end-to-end path). */
typedef struct {
  int64_t n_clients;
  const int64_t* n_samples; /* [n_clients], host, copied at init */
  int32_t feature_dim;      /* 784, 3072, 3920 or 80 */
  const void* x;
  const int32_t* y;
  int32_t on_device;
} fl_population;

/* Device-time statistics of the last round on this rank (CUDA events on the ctx stream). */
typedef struct {
  double round_ms;      /* fl_round entry (plan on host) to θ_new resident on this GPU */
  double place_ms;      /* host placement + packing (wall) */
  double stage_ms;      /* cohort gather / host->device staging */
  double train_ms;      /* local SGD of this rank's clients (device) */
  double agg_ms;        /* fused per-GPU accumulation + (NCCL reduce) + finalize */
  double allreduce_ms;  /* NCCL part of agg_ms (0 without a communicator) */
  double client_updates_per_s; /* clients_total / round_ms_max */
  int64_t clients_total, clients_local;
  int64_t samples_total, samples_local;
  int64_t steps_local;  /* Σ E·m over this rank's clients */
  int64_t waves;        /* max E·m over this rank's clients (critical path in SGD steps) */
  int64_t h2d_bytes;    /* host->device bytes copied this round */
  int64_t kernels;      /* kernel launches this round */
  double train_end_ms;  /* fl_round entry to the end of this rank's local SGD (device) */
  /* Over ranks (all-gathered through the communicator; equal to this rank's values without one): */
  double round_ms_max;  /* the round time: max over ranks of round_ms */
  double train_end_ms_min, train_end_ms_max;
  double timedelta_ms;  /* "timedelta workers": train_end_ms_max − train_end_ms_min */
  int64_t xfer_bytes;   /* bytes this rank sent to other ranks' memory in the aggregation
                           (peer / unaggregated modes; NCCL: 8·(P_pad+1)·2·(W−1)/W, ring estimate) */
  int32_t sm_count;     /* SMs this rank's kernels may use (its green-context partition) */
} fl_round_stats;

uint32_t fl_abi_version(void);

/* Canonical parameter count P of a model (torch state_dict order, §8c.2 of SURVEY):
 * logreg 7,850; CNN 2,156,490; speech 3,993,507; LSTM 819,920.  0 if unknown. */
int64_t fl_n_params(int32_t model);

/* ---- host-only planning (no device needed) -------------------------------- */
/* Placement (§5): cohort_ids[n_cohort] distinct ids < n_clients; n_samples[n_clients].
 * Writes out_ids[n_cohort] grouped by worker in assignment order (largest first for
 * SRR/BU/LB) and out_off[world_size+1] CSR offsets.  lb_coef = (a,b,c,d) for LB,
 * ignored otherwise.  FL_ERR_INVALID on unknown/duplicate id, n_cohort > n_clients,
 * world_size < 1, batch_size < 1, n_samples < 1 of a cohort member, LB without coef. */
fl_status fl_place_plan(int32_t policy, const int64_t* cohort_ids, int64_t n_cohort,
                        const int64_t* n_samples, int64_t n_clients, int32_t batch_size,
                        int32_t world_size, const double* lb_coef,
                        int64_t* out_ids, int64_t* out_off);

/* LB's time model: least-squares fit of Eq. 3
 * y = a·x + b·ln(c·x) + d to n >= 4 records (x[i] = batches m >= 1 of a trained
 * client, y[i] = its measured training time, any unit).  Because
 * b·ln(c·x) + d = b·ln x + (b·ln c + d), c is not identifiable: the fit
 * returns c = 1 and the exact least-squares minimiser over (a, b, d) (Householder
 * QR).  It is accepted if a >= 0 and it predicts > 0 over [min x, max x];
 * otherwise the fallback is the line a·x + d with a >= 0, else the mean.
 * coef_out[4] = (a, b, c, d); *kind_out = 0 Eq. 3, 1 line, 2 constant (nullable);
 * *mse_out = mean squared residual (nullable).  FL_ERR_INVALID if n < 4, any x < 1, or any
 * x / y not finite. */
fl_status fl_lb_fit(const double* x, const double* y, int64_t n, double* coef_out, int32_t* kind_out,
                    double* mse_out);

/* Ragged packer for one worker list ids[n]: seg_off[n+1] prefix sums of
 * n_samples in list order; steps[n] = E·ceil(n_k/B). */
fl_status fl_pack_plan(const int64_t* ids, int64_t n, const int64_t* n_samples, int64_t n_clients,
                       int32_t batch_size, int32_t local_epochs, int64_t* seg_off, int64_t* steps);

/* ---- context ---------------------------------------------------------------- */
/* Writes 128 bytes of a fresh NCCL unique id (call on rank 0, broadcast to others). */
fl_status fl_nccl_unique_id(uint8_t* out128);

/* global_params: host float32[n_params] in canonical layout; n_params must equal
 * fl_n_params(cfg->model).  Allocates device state for the population and the
 * largest cohort share this rank can receive (n_clients). */
fl_status fl_round_init(const fl_config* cfg, const fl_population* pop,
                        const float* global_params, int64_t n_params, fl_ctx** out);

/* Push-based placement of a round's cohort.  Stores the plan in
 * the ctx; out_ids / out_off may be NULL. */
fl_status fl_place(fl_ctx* ctx, const int64_t* cohort_ids, int64_t n_cohort, int32_t policy,
                   const double* lb_coef, int64_t* out_ids, int64_t* out_off);

/* Local SGD of this rank's share of the last plan (stream-ordered, asynchronous).
 * round_index keys the shuffle (A5).  FL_ERR_STATE if no plan. */
fl_status fl_train_clients(fl_ctx* ctx, int32_t round_index);

/* Fused per-GPU weighted accumulation S_g = Σ n_k(θ_k − θ_g) (fp64), NCCL allreduce
 * of [S_g ‖ N_g] when world_size > 1, θ_new = fp32(θ_g + S/N) (Eq. 1-2 in delta form,
 * reading A2).  θ_new becomes the ctx's θ_g.  out_params: nullable host float32[P]
 * (canonical layout, synchronous copy); out_total_samples: nullable. */
fl_status fl_aggregate(fl_ctx* ctx, float* out_params, int64_t* out_total_samples);

/* fl_aggregate with the copy of θ_new only ENQUEUED on the ctx stream: the call returns
 * without waiting, so the host can place and issue the next round while this one runs on
 * the device (rounds are stream-ordered: the next round reads this θ_new on the device).
 * out_params: nullable; else page-locked host float32[P] (cudaHostAlloc / cudaHostRegister /
 * torch pin_memory), FL_ERR_INVALID for pageable memory.  Its contents are valid after
 * fl_synchronize (or any later synchronising call) and must not be reused before. */
fl_status fl_aggregate_async(fl_ctx* ctx, float* out_params, int64_t* out_total_samples);

/* Block until all work issued on the ctx (rounds, copies) has completed. */
fl_status fl_synchronize(fl_ctx* ctx);

/* fl_place + fl_train_clients + fl_aggregate, timed; stats nullable.  Asynchronous
 * with respect to the host except for the stats event reads (it synchronises the
 * ctx stream when stats != NULL).  With a communicator, stats != NULL makes the call
 * gather every rank's times (round_ms_max, timedelta_ms): all ranks must then pass
 * stats != NULL for that round. */
fl_status fl_round(fl_ctx* ctx, const int64_t* cohort_ids, int64_t n_cohort, int32_t policy,
                   const double* lb_coef, int32_t round_index, fl_round_stats* stats);

/* ---- parity / test entry points ---------------------------------------------- */
/* Weighted FedAvg of K arbitrary fp32 vectors of length P (device pointers):
 * out = fp32(θ_g + Σ n_k(θ_k − θ_g) / Σ n_k), fp64 accumulation in index order k.
 * theta_k: device float32[K][P]; n: host int64[K] (>= 1); theta_g, out: device float32[P]. */
fl_status fl_fedavg_vectors(fl_ctx* ctx, const float* theta_k, const int64_t* n, int64_t K,
                            int64_t P, const float* theta_g, float* out);

/* This rank's local plan: ids[n_local] (execution order = plan order), seg_off[n_local+1],
 * steps[n_local]; any pointer may be NULL; *n_local always written. */
fl_status fl_get_local_plan(fl_ctx* ctx, int64_t* ids, int64_t* seg_off, int64_t* steps,
                            int64_t* n_local);

/* θ_k of a locally trained client after fl_train_clients (host float32[P], canonical). */
fl_status fl_get_client_params(fl_ctx* ctx, int64_t client_id, float* out);

/* Current θ_g (host float32[P], canonical) / replace it. */
fl_status fl_get_global_params(fl_ctx* ctx, float* out);
fl_status fl_set_global_params(fl_ctx* ctx, const float* params);

/* LB timing records ("collects the training time of each client").  With
 * records on, fl_train_clients records a CUDA event on a client's group stream after
 * the wave in which its last SGD step runs; fl_get_client_times then returns, per
 * local client in plan order, ids[i], m[i] = ceil(n/B) and t_ms[i] = device time from
 * the end of staging to that event (the client's completion time on this GPU: clients
 * train concurrently, so this is the time a client of that size costs the GPU's round).
 * Arrays have room for n_local = clients placed on this rank; blocks until the round's
 * training is done.  FL_ERR_STATE if no round was trained with records on. */
fl_status fl_set_timing_records(fl_ctx* ctx, int32_t on);
fl_status fl_get_client_times(fl_ctx* ctx, int64_t* ids, int64_t* m, double* t_ms, int64_t* n_local);

/* Stats of the last fl_round.  With a communicator this is a collective call (the
 * over-ranks fields are all-gathered): every rank must call it. */
fl_status fl_get_stats(fl_ctx* ctx, fl_round_stats* out);

/* Per-kernel-class device time of the last round, for roofline reports.  Off by default:
 * fl_set_profiling(ctx, 1) brackets every launch with CUDA events on the ctx stream (adds
 * a small gap between launches; do not time throughput with it on).  kind indexes the
 * classes 0 .. n-1 (names: pack, conv1_fwd, ..., fedavg_accum); FL_ERR_INVALID past the
 * end.  flops / bytes are the ALGORITHMIC work of those launches. */
typedef struct {
  char name[32];
  double ms;        /* Σ of launch durations */
  int64_t launches;
  double flops;     /* Σ algorithmic FLOPs */
  double bytes;     /* Σ algorithmic HBM bytes */
} fl_kernel_stats;
fl_status fl_set_profiling(fl_ctx* ctx, int32_t on);
fl_status fl_get_kernel_stats(fl_ctx* ctx, int32_t kind, fl_kernel_stats* out);

/* ---- peer-memory aggregation (agg_mode FL_AGG_PEER / FL_AGG_UNAGGREGATED) ----------- */
/* A rank's peer blob: FL_PEER_BLOB_BYTES opaque bytes (process id, device, CUDA IPC handles and
 * addresses of this ctx's partial buffer S, θ_g, signal words and the unaggregated receive
 * buffer).  Every rank exports one; the caller all-gathers them (e.g. torch.distributed) and
 * passes the array [world_size][FL_PEER_BLOB_BYTES] in rank order to fl_peer_connect, which maps
 * the peers' buffers (IPC across processes, plain pointers for ranks in one process) and enables
 * peer access across devices.  Ranks sharing one device must run on disjoint SM partitions
 * (sm_count), because the aggregation kernel of one rank waits on the device for its peers';
 * FL_ERR_INVALID otherwise.  Such a process should run with CUDA_MODULE_LOADING=EAGER (a lazily
 * loaded kernel variant can stall behind a spinning peer) and CUDA_DEVICE_MAX_CONNECTIONS=32 (the
 * ranks' streams otherwise share 8 hardware queues and serialise).  fl_peer_export needs the largest cohort size this rank will
 * aggregate as a server (max_clients, for the unaggregated receive buffer; ignored elsewhere).
 * Collective in effect: a round's fl_aggregate completes only when every rank ran its own. */
#define FL_PEER_BLOB_BYTES 512
fl_status fl_peer_export(fl_ctx* ctx, int64_t max_clients, uint8_t* out_blob);
fl_status fl_peer_connect(fl_ctx* ctx, const uint8_t* blobs, int32_t world_size);

/* The cudaStream_t the ctx launches on (for the caller's event timing). */
void* fl_get_stream(fl_ctx* ctx);

const char* fl_last_error(const fl_ctx* ctx); /* ctx-owned string; "" if none; NULL ctx ok */
void fl_round_destroy(fl_ctx* ctx);           /* NULL ok */

#ifdef __cplusplus
}
#endif
#endif /* FL_B200_H */
