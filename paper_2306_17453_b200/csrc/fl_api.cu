// fl_api.cu — the C-ABI (include/fl.h): context, staging, wave scheduling, aggregation.
//
// Round = place (host, §5) -> pack/stage (host tables + K3 gather) -> local SGD of every
// local client as waves of grouped kernels (a4-a7) -> fused fp64 accumulation (K1) ->
// NCCL allreduce of [S ‖ N] across ranks (a9) -> finalize (K2).  PAPER.md §4.1-4.4,
// Eq. 1-2; SURVEY.md §3.3.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <unistd.h>
#include <nccl.h>  // types only; the library is dlopen'ed when world_size > 1
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/fl.h"
#include "../../include/fl_debug.h"
#include "fl_host.h"
#include "fl_internal.h"

namespace flb {

const char* const kKindName[K_NKINDS] = {
    "pack", "conv1_fwd", "pool1", "conv2_fwd", "pool2", "fc1_fwd", "head_fc2_ce", "fc1_dx", "unpool2",
    "fc1_dw_sgd", "conv2_dx", "unpool1", "conv2_dw", "conv2_dw_reduce_sgd", "conv1_dw", "conv1_dw_reduce_sgd",
    "logreg_client", "fedavg_accum", "lstm_step"};

// ---------------------------------------------------------------- layouts
static int64_t up32(int64_t x) { return (x + 31) / 32 * 32; }

bool make_layout(int model, Layout* L) {
  L->model = model;
  L->canon_of.clear();
  if (model == FL_MODEL_LOGREG) {
    L->P = 7850;
    L->P_pad = up32(7850);
    L->D_in = 784;
    L->D_pack = 784;
    L->canon_of.assign((size_t)L->P_pad, -1);
    for (int64_t i = 0; i < 7850; ++i) L->canon_of[(size_t)i] = i;
    return true;
  }
  if (model == FL_MODEL_CHAR_LSTM) return lstm_layout(L);
  if (model != FL_MODEL_CNN_CIFAR && model != FL_MODEL_CNN_SPEECH) return false;
  CnnDims& d = L->d;
  if (model == FL_MODEL_CNN_CIFAR) { d.cin = 3; d.H0 = 32; d.W0 = 32; d.HID = 512; d.NCLS = 10; }
  else { d.cin = 1; d.H0 = 40; d.W0 = 98; d.HID = 256; d.NCLS = 35; }
  // pixels padded to 4 channels (one 16-byte TMA/UMMA column) for the CIFAR tensor-core path;
  // the 1-channel speech input stays unpadded (its FP32 conv1 would do 4x the work otherwise)
  d.cpad = model == FL_MODEL_CNN_CIFAR ? 4 : 1; d.C1 = 32; d.C2 = 64;
  d.H1 = d.H0 / 2; d.W1 = d.W0 / 2; d.H2 = d.H1 / 2; d.W2 = d.W1 / 2;
  d.F = d.C2 * d.H2 * d.W2;
  L->D_in = d.cin * d.H0 * d.W0;
  L->D_pack = d.cpad * d.H0 * d.W0;
  // canonical (torch) offsets
  const int64_t c_c1w = 0, c_c1b = c_c1w + (int64_t)d.C1 * d.cin * 25, c_c2w = c_c1b + d.C1,
                c_c2b = c_c2w + (int64_t)d.C2 * d.C1 * 25, c_f1w = c_c2b + d.C2, c_f1b = c_f1w + (int64_t)d.HID * d.F,
                c_f2w = c_f1b + d.HID, c_f2b = c_f2w + (int64_t)d.NCLS * d.HID, c_end = c_f2b + d.NCLS;
  L->P = c_end;
  int64_t o = 0;
  L->o_c1w = o; o = up32(o + (int64_t)d.C1 * 25 * d.cpad);
  L->o_c1b = o; o = up32(o + d.C1);
  L->o_c2w = o; o = up32(o + (int64_t)d.C2 * 25 * d.C1);
  L->o_c2b = o; o = up32(o + d.C2);
  L->o_f1w = o; o = up32(o + (int64_t)d.HID * d.F);
  L->o_f1b = o; o = up32(o + d.HID);
  L->o_f2w = o; o = up32(o + (int64_t)d.NCLS * d.HID);
  L->o_f2b = o; o = up32(o + d.NCLS);
  L->P_pad = o;
  std::vector<int64_t>& m = L->canon_of;
  m.assign((size_t)L->P_pad, -1);
  for (int oc = 0; oc < d.C1; ++oc)
    for (int t = 0; t < 25; ++t)
      for (int c = 0; c < d.cin; ++c) m[(size_t)(L->o_c1w + ((int64_t)oc * 25 + t) * d.cpad + c)] = c_c1w + ((int64_t)oc * d.cin + c) * 25 + t;
  for (int oc = 0; oc < d.C1; ++oc) m[(size_t)(L->o_c1b + oc)] = c_c1b + oc;
  for (int oc = 0; oc < d.C2; ++oc)
    for (int t = 0; t < 25; ++t)
      for (int c = 0; c < d.C1; ++c) m[(size_t)(L->o_c2w + ((int64_t)oc * 25 + t) * d.C1 + c)] = c_c2w + ((int64_t)oc * d.C1 + c) * 25 + t;
  for (int oc = 0; oc < d.C2; ++oc) m[(size_t)(L->o_c2b + oc)] = c_c2b + oc;
  // fc1 columns: internal (h,w,c) order of the NHWC pooled map, canonical (c,h,w)
  for (int n = 0; n < d.HID; ++n)
    for (int h = 0; h < d.H2; ++h)
      for (int w = 0; w < d.W2; ++w)
        for (int c = 0; c < d.C2; ++c)
          m[(size_t)(L->o_f1w + (int64_t)n * d.F + ((int64_t)h * d.W2 + w) * d.C2 + c)] =
              c_f1w + (int64_t)n * d.F + ((int64_t)c * d.H2 + h) * d.W2 + w;
  for (int n = 0; n < d.HID; ++n) m[(size_t)(L->o_f1b + n)] = c_f1b + n;
  for (int64_t i = 0; i < (int64_t)d.NCLS * d.HID; ++i) m[(size_t)(L->o_f2w + i)] = c_f2w + i;
  for (int q = 0; q < d.NCLS; ++q) m[(size_t)(L->o_f2b + q)] = c_f2b + q;
  return true;
}

CnnBufs cnn_group_view(const CnnBufs& b, const CnnDims& d, int B, int64_t base_client, int64_t nclients, int g,
                       int64_t per_group_z, int64_t part2_z_floats, int64_t part1_z_floats) {
  CnnBufs v = b;
  const int64_t s0 = base_client * B;
  const int64_t hw0 = (int64_t)d.H0 * d.W0, hw1 = (int64_t)d.H1 * d.W1, hw2 = (int64_t)d.H2 * d.W2;
  v.a1 = b.a1 ? b.a1 + s0 * hw0 * d.C1 : nullptr;  // full-resolution planes: SIMT path only
  v.dY1 = b.dY1 ? b.dY1 + s0 * hw0 * d.C1 : nullptr;
  v.p1 = b.p1 + s0 * hw1 * d.C1;
  v.am1 = b.am1 + s0 * hw1 * d.C1;
  v.dp1 = b.dp1 + s0 * hw1 * d.C1;
  v.a2 = b.a2 + s0 * hw1 * d.C2;
  v.dY2 = b.dY2 + s0 * hw1 * d.C2;
  v.p2 = b.p2 + s0 * hw2 * d.C2;
  v.am2 = b.am2 + s0 * hw2 * d.C2;
  v.dp2 = b.dp2 + s0 * hw2 * d.C2;
  v.h = b.h + s0 * d.HID;
  v.dh = b.dh + s0 * d.HID;
  v.dz = b.dz + s0 * d.NCLS;
  v.slots = nclients * B;
  v.clients = nclients;
  v.part2 = b.part2 + (int64_t)g * per_group_z * part2_z_floats;
  v.part1 = b.part1 + (int64_t)g * per_group_z * part1_z_floats;
  v.part2_tc_cap = per_group_z;
  v.part1_tc_cap = per_group_z;
  v.fc1_part = b.fc1_part + (int64_t)g * b.fc1_part_floats;
  return v;
}

}  // namespace flb

using namespace flb;

// ---------------------------------------------------------------- NCCL (dlopen)
namespace {
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*getVersion)(int*) = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
  bool load() {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
    commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
    allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    errStr = (decltype(errStr))dlsym(h, "ncclGetErrorString");
    allGather = (decltype(allGather))dlsym(h, "ncclAllGather");
    commCount = (decltype(commCount))dlsym(h, "ncclCommCount");
    getVersion = (decltype(getVersion))dlsym(h, "ncclGetVersion");
    return getUniqueId && commInitRank && allReduce && commDestroy && allGather;
  }
};
Nccl g_nccl;

// Grow-only device buffers.  A replaced buffer is retired to `grave` and freed when the context
// is destroyed, not here: cudaFree synchronises the whole device, so a rank that grows a buffer
// mid-run would wait for every other context's kernels — including a peer rank's aggregation
// kernel that is itself waiting for this rank (two ranks in one process, f3/f4), a stall of up to
// a second per growth.  Growth allocates 1/8 headroom so share changes rarely trigger it.
template <class T>
cudaError_t grow_dev(std::vector<void*>& grave, T*& p, int64_t& cap, int64_t need) {
  if (need <= cap && p) return cudaSuccess;
  if (p) grave.push_back(p);
  p = nullptr;
  if (cap > 0) need += need / 8;
  int64_t n = std::max<int64_t>(need, 1);
  cudaError_t e = cudaMalloc((void**)&p, sizeof(T) * (size_t)n);
  cap = e == cudaSuccess ? n : 0;
  return e;
}
// Green contexts (CUDA driver API through the runtime's entry-point table, no -lcuda):
// an SM partition of the device whose streams only run on its SMs (include/fl.h sm_count).
template <class F>
F drv(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return nullptr;
  return (F)fn;
}
struct GreenPart {
  CUgreenCtx g = nullptr;
  int sms = 0;
  CUresult (*stream_create)(CUstream*, CUgreenCtx, unsigned, int) = nullptr;
};
// s > 0: the first partition of >= s SMs; s < 0: the remainder after splitting off >= -s SMs
bool green_partition(int device, int s, GreenPart* out, std::string* err) {
  auto devGet = drv<CUresult (*)(CUdevice*, int)>("cuDeviceGet");
  auto getRes = drv<CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType)>("cuDeviceGetDevResource");
  auto split = drv<CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned)>(
      "cuDevSmResourceSplitByCount");
  auto gen = drv<CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned)>("cuDevResourceGenerateDesc");
  auto gcreate = drv<CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned)>("cuGreenCtxCreate");
  out->stream_create = drv<CUresult (*)(CUstream*, CUgreenCtx, unsigned, int)>("cuGreenCtxStreamCreate");
  if (!devGet || !getRes || !split || !gen || !gcreate || !out->stream_create) {
    *err = "driver has no green-context entry points";
    return false;
  }
  CUdevice dev;
  CUdevResource all, part, rem;
  unsigned nb = 1;
  CUresult r;
  if ((r = devGet(&dev, device)) != CUDA_SUCCESS || (r = getRes(dev, &all, CU_DEV_RESOURCE_TYPE_SM)) != CUDA_SUCCESS ||
      (r = split(&part, &nb, &all, &rem, 0, (unsigned)(s > 0 ? s : -s))) != CUDA_SUCCESS || nb != 1) {
    *err = "cannot split the device's SMs (CUresult " + std::to_string((int)r) + ")";
    return false;
  }
  CUdevResource* use = s > 0 ? &part : &rem;
  if (use->sm.smCount == 0) {
    *err = "empty SM partition";
    return false;
  }
  CUdevResourceDesc desc;
  if ((r = gen(&desc, use, 1)) != CUDA_SUCCESS || (r = gcreate(&out->g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM)) != CUDA_SUCCESS) {
    *err = "cuGreenCtxCreate failed (CUresult " + std::to_string((int)r) + ")";
    return false;
  }
  out->sms = (int)use->sm.smCount;
  return true;
}

// peer blob (include/fl.h FL_PEER_BLOB_BYTES): what a rank tells the others about its buffers
struct PeerBlob {
  uint64_t magic;
  int32_t pid, device, sm_count, world, rank, T;
  int64_t P_pad, recv_cap;
  uint64_t ptr[4];                 // S, theta, sig, recv (valid in the exporting process)
  cudaIpcMemHandle_t h[4];
};
static_assert(sizeof(PeerBlob) <= FL_PEER_BLOB_BYTES, "peer blob too large");
constexpr uint64_t kPeerMagic = 0x464c50454552310aull;  // "FLPEER1\n"
constexpr int64_t kPeerTile = 8192;                    // parameters per aggregation tile
}  // namespace

struct fl_ctx {
  fl_config cfg{};
  Layout L;
  int64_t n_pop = 0;
  std::vector<int64_t> n_samples, pop_off;
  const void* x = nullptr;
  const int32_t* y = nullptr;
  bool pop_dev = false, host_registered = false;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  ncclComm_t comm = nullptr;

  float* d_theta = nullptr;  // θ_g, internal layout [P_pad]
  int64_t* d_canon_of = nullptr;
  float* d_canon = nullptr;  // scratch [P]
  float* d_slots = nullptr;
  int64_t slots_cap = 0;
  double* d_S = nullptr;  // [P_pad + 1] (world > 1)

  // plan
  bool have_plan = false, trained = false, failed = false;
  std::vector<int64_t> plan_ids, plan_off, local_ids;  // local_ids in plan order
  std::vector<int64_t> exec;                           // exec position -> index into local_ids
  std::vector<int64_t> exec_ids;                       // client id of exec position e (last trained round)
  std::vector<int64_t> steps_exec, n_exec, pseg;
  int64_t N_total = 0, N_local = 0, K_total = 0;

  // staging
  float* d_xpack = nullptr;
  int64_t xpack_cap = 0;
  int32_t* d_ypack = nullptr;
  int64_t ypack_cap = 0;
  // host-population staging, double-buffered across rounds: round r copies into buffer r % 2
  // while round r−1 may still run (only its packs wait for round r−1, ev_start)
  float* d_stage = nullptr;   // this round's buffer (one of d_stage2)
  int32_t* d_ystage = nullptr;
  float* d_stage2[2] = {nullptr, nullptr};
  int64_t stage_cap2[2] = {0, 0};
  int32_t* d_ystage2[2] = {nullptr, nullptr};
  int64_t ystage_cap2[2] = {0, 0};
  cudaEvent_t ev_sfree[2] = {nullptr, nullptr};  // recorded after the last pack reading buffer b
  int stage_par = 0;
  int64_t* d_src_row = nullptr;
  int64_t src_cap = 0;
  int64_t* d_n = nullptr;
  int64_t n_cap = 0;
  int32_t* d_steps = nullptr;
  int64_t steps_cap = 0;
  int64_t* d_slot_off = nullptr;
  int64_t slot_off_cap = 0;
  int64_t sidx_cap = 0, bs_cap = 0, bpre_cap = 0;
  WaveSched ws;
  CnnBufs cb;
  LstmBufs lb;
  int64_t cb_slots_cap = 0, cb_part_cap = 0;

  // pinned host staging of the per-round tables: a ring of two buffers, so issuing round r
  // waits (ev_tab[r % 2]) only for the table copies of round r - 2
  char* h_tab[2] = {nullptr, nullptr};
  size_t h_tab_cap[2] = {0, 0};
  bool tab_pending[2] = {false, false};
  cudaEvent_t ev_tab[2] = {nullptr, nullptr};
  int tab_i = 0;
  double tab_wait_ms = 0.0;
  // per-rank [round_ms, train_end_ms] gathered over the communicator for the round stats
  double* h_rstat = nullptr;  // pinned [2·world]
  double* d_rstat = nullptr;  // device [2 + 2·world]

  cudaEvent_t ev_entry = nullptr, ev_start = nullptr, ev_staged = nullptr, ev_trained = nullptr,
              ev_agg0 = nullptr, ev_acc1 = nullptr, ev_ar0 = nullptr, ev_ar1 = nullptr, ev_end = nullptr;
  double place_ms = 0.0;
  int64_t kernels = 0, h2d = 0, train_launches = 0;
  fl_round_stats stats{};
  KProf prof;
  std::string err;
  // concurrent client groups (CNN): streams forked from / joined into st
  // Measured on C2 (scripts/group_sweep.py): 4 solo + 2 shared groups is best; more than 8
  // streams in total alias onto the device's 8 hardware queues and serialise.
  int ngroups = 2;  // round-robin groups (FL_GROUPS)
  int nsolo = 4;    // longest clients given their own high-priority group (FL_SOLO)
  // SMs the bulk groups' persistent kernels leave free for the solo (critical-path) streams
  // when solo groups exist (FL_RESERVE_SMS; measured: 64 -> C2 -3%; after the 8-warp fc1
  // backward 32 is C2-neutral and 4% faster on a 400-client C3-law cohort)
  int reserve_sms = 32;
  // SMs a solo group's persistent kernels may occupy (FL_SOLO_SMS)
  int solo_sms = 148;
  std::vector<cudaStream_t> gstream;  // [nsolo high-priority | ngroups normal]
  std::vector<cudaEvent_t> ev_join;
  cudaEvent_t ev_fork = nullptr;
  int64_t part_group_z = 0;
  // LB timing records (fl_set_timing_records): one event per (group, wave) in which some
  // client's last step runs; rec_of_exec[e] = index into rec_ev of exec position e's event
  bool rec_on = false, rec_valid = false;
  std::vector<cudaEvent_t> rec_ev;
  std::vector<int64_t> rec_of_exec;
  // pipelined staging of a host population: copies + pack of chunk q run on cst and
  // complete on ev_chunk[q]; the waves of local step t >= chunk_t0[q] wait for it
  cudaStream_t cst = nullptr;
  cudaStream_t pst = nullptr;  // high-priority pack stream: a pack kernel waiting for SMs never stalls the copies
  std::vector<cudaEvent_t> ev_chunk, ev_copy;
  // SM partition (cfg.sm_count): green context whose streams run on n_sms SMs only
  GreenPart green;
  int n_sms = 148;
  // peer-memory aggregation (FL_AGG_PEER / FL_AGG_UNAGGREGATED)
  bool peer_on = false;
  PeerArgs peer{};
  std::vector<void*> ipc_opened;             // peer buffers mapped with cudaIpcOpenMemHandle
  std::vector<void*> grave;                  // replaced device buffers, freed at destroy (grow_dev)
  unsigned long long* d_sig = nullptr;       // [(FL_MAX_PEERS + 1) · T] signal words
  int peer_T = 0;
  float* d_recv = nullptr;                   // server (rank 0) receive buffer, unaggregated mode
  int64_t recv_cap = 0;
  int64_t* d_dst_row = nullptr;              // [K] receive row of each exec slot (unaggregated)
  int64_t dst_cap = 0;
  int64_t* d_nplan = nullptr;                // server: [K_total] n of each received row
  int64_t nplan_cap = 0;
  unsigned int* d_ctr = nullptr;             // last-CTA counters of the push / broadcast kernels
  unsigned long long agg_seq = 0;
  int64_t xfer_bytes = 0;
};

// ---------------------------------------------------------------- error helpers
static fl_status set_err(fl_ctx* c, fl_status s, const char* fmt, ...) {
  if (!c) return s;
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  c->err = buf;
  if (s == FL_ERR_CUDA || s == FL_ERR_NCCL || s == FL_ERR_OOM) c->failed = true;
  return s;
}

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return set_err(c, e_ == cudaErrorMemoryAllocation ? FL_ERR_OOM : FL_ERR_CUDA, "%s: %s (%s:%d)", \
                     #call, cudaGetErrorString(e_), __FILE__, __LINE__);                          \
  } while (0)

#define CKL()                                                                                     \
  do {                                                                                            \
    cudaError_t e_ = cudaGetLastError();                                                          \
    if (e_ != cudaSuccess)                                                                        \
      return set_err(c, FL_ERR_CUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

static bool model_supported(int m) {
  return m == FL_MODEL_LOGREG || m == FL_MODEL_CNN_CIFAR || m == FL_MODEL_CNN_SPEECH || m == FL_MODEL_CHAR_LSTM;
}

extern "C" {

uint32_t fl_abi_version(void) { return FL_ABI_VERSION; }

int64_t fl_n_params(int32_t model) {
  switch (model) {
    case FL_MODEL_LOGREG: return 7850;
    case FL_MODEL_CNN_CIFAR: return 2156490;
    case FL_MODEL_CNN_SPEECH: return 3993507;
    case FL_MODEL_CHAR_LSTM: return 819920;
  }
  return 0;
}

fl_status fl_place_plan(int32_t policy, const int64_t* cohort_ids, int64_t n_cohort, const int64_t* n_samples,
                        int64_t n_clients, int32_t batch_size, int32_t world_size, const double* lb_coef,
                        int64_t* out_ids, int64_t* out_off) {
  if (!cohort_ids && n_cohort > 0) return FL_ERR_INVALID;
  if (!n_samples || !out_off || (!out_ids && n_cohort > 0)) return FL_ERR_INVALID;
  return (fl_status)place(policy, cohort_ids, n_cohort, n_samples, n_clients, batch_size, world_size, lb_coef,
                          out_ids, out_off);
}

fl_status fl_lb_fit(const double* x, const double* y, int64_t n, double* coef_out, int32_t* kind_out,
                    double* mse_out) {
  if (!x || !y || !coef_out) return FL_ERR_INVALID;
  const int kind = lb_fit(x, y, n, coef_out, mse_out);
  if (kind < 0) return FL_ERR_INVALID;
  if (kind_out) *kind_out = kind;
  return FL_OK;
}

fl_status fl_pack_plan(const int64_t* ids, int64_t n, const int64_t* n_samples, int64_t n_clients, int32_t batch_size,
                       int32_t local_epochs, int64_t* seg_off, int64_t* steps) {
  if ((!ids && n > 0) || !n_samples) return FL_ERR_INVALID;
  return (fl_status)pack(ids, n, n_samples, n_clients, batch_size, local_epochs, seg_off, steps);
}

fl_status fl_nccl_unique_id(uint8_t* out128) {
  if (!out128) return FL_ERR_INVALID;
  if (!g_nccl.load()) return FL_ERR_NCCL;
  ncclUniqueId id;
  if (g_nccl.getUniqueId(&id) != ncclSuccess) return FL_ERR_NCCL;
  memcpy(out128, id.internal, 128);
  return FL_OK;
}

const char* fl_last_error(const fl_ctx* c) { return c ? c->err.c_str() : ""; }

void* fl_get_stream(fl_ctx* c) { return c ? (void*)c->st : nullptr; }

void fl_round_destroy(fl_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->cfg.device);
  if (c->st) cudaStreamSynchronize(c->st);
  if (c->comm && g_nccl.commDestroy) g_nccl.commDestroy(c->comm);
  void* ptrs[] = {c->d_theta, c->d_canon_of, c->d_canon, c->d_slots, c->d_S, c->d_xpack, c->d_ypack, c->d_stage2[0],
                  c->d_ystage2[0], c->d_stage2[1], c->d_ystage2[1], c->d_src_row, c->d_n, c->d_steps, c->d_slot_off, c->ws.d_sidx, c->ws.d_bs, c->ws.d_bpre,
                  c->cb.a1, c->cb.p1, c->cb.a2, c->cb.p2, c->cb.h, c->cb.dh, c->cb.am1, c->cb.am2, c->cb.dp2,
                  c->cb.dY2, c->cb.dp1, c->cb.dY1, c->cb.part1, c->cb.part2, c->cb.xg, c->cb.fc1_part,
                  c->cb.dz, c->lb.xp, c->lb.G0, c->lb.G1, c->lb.dpre, c->lb.C0, c->lb.C1, c->lb.H0, c->lb.H1,
                  c->lb.dX, c->lb.E, c->lb.dE, c->lb.dhT};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  for (void* p : c->grave) cudaFree(p);
  void* pptrs[] = {c->d_sig, c->d_recv, c->d_dst_row, c->d_nplan, c->d_ctr};
  for (void* p : pptrs)
    if (p) cudaFree(p);
  for (int i = 0; i < 2; ++i)
    if (c->h_tab[i]) cudaFreeHost(c->h_tab[i]);
  if (c->h_rstat) cudaFreeHost(c->h_rstat);
  if (c->d_rstat) cudaFree(c->d_rstat);
  cudaEvent_t evs[] = {c->ev_entry, c->ev_start, c->ev_staged, c->ev_trained, c->ev_agg0,
                       c->ev_acc1, c->ev_ar0, c->ev_ar1, c->ev_end, c->ev_tab[0], c->ev_tab[1],
                       c->ev_sfree[0], c->ev_sfree[1]};
  for (cudaEvent_t e : evs)
    if (e) cudaEventDestroy(e);
  if (c->host_registered) cudaHostUnregister((void*)c->x);
  for (cudaStream_t s : c->gstream)
    if (s) cudaStreamDestroy(s);
  for (cudaEvent_t e : c->ev_join)
    if (e) cudaEventDestroy(e);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  for (cudaEvent_t e : c->rec_ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ev_chunk)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ev_copy)
    if (e) cudaEventDestroy(e);
  if (c->cst) cudaStreamDestroy(c->cst);
  if (c->pst) cudaStreamDestroy(c->pst);
  if (c->own_stream && c->st) cudaStreamDestroy(c->st);
  if (c->green.g) {
    auto gdestroy = drv<CUresult (*)(CUgreenCtx)>("cuGreenCtxDestroy");
    if (gdestroy) gdestroy(c->green.g);
  }
  delete c;
}

fl_status fl_round_init(const fl_config* cfg, const fl_population* pop, const float* global_params, int64_t n_params,
                        fl_ctx** out) {
  if (!cfg || !pop || !global_params || !out) return FL_ERR_INVALID;
  *out = nullptr;
  if (cfg->abi_version != FL_ABI_VERSION) return FL_ERR_INVALID;
  if (cfg->batch_size < 1 || cfg->local_epochs < 1 || !(cfg->lr >= 0.f) || cfg->min_samples < 1) return FL_ERR_INVALID;
  if (cfg->world_size < 1 || cfg->rank < 0 || cfg->rank >= cfg->world_size) return FL_ERR_INVALID;
  if (cfg->agg_mode < FL_AGG_NCCL || cfg->agg_mode > FL_AGG_UNAGGREGATED) return FL_ERR_INVALID;
  if (cfg->world_size > FL_MAX_PEERS && cfg->agg_mode != FL_AGG_NCCL) return FL_ERR_INVALID;
  // NCCL aggregation across ranks needs the communicator's id (world 1 + id: a 1-rank comm)
  if (cfg->world_size > 1 && cfg->agg_mode == FL_AGG_NCCL && !cfg->nccl_unique_id) return FL_ERR_INVALID;
  if (cfg->sm_count != 0 && cfg->stream) return FL_ERR_INVALID;  // a borrowed stream cannot be partitioned
  if (fl_n_params(cfg->model) == 0) return FL_ERR_INVALID;
  if (n_params != fl_n_params(cfg->model)) return FL_ERR_INVALID;
  if (!model_supported(cfg->model)) return FL_ERR_UNSUPPORTED;
  if (pop->n_clients < 1 || !pop->n_samples || !pop->x || !pop->y) return FL_ERR_INVALID;
  fl_ctx* c = new fl_ctx();
  c->cfg = *cfg;
  make_layout(cfg->model, &c->L);
  // the LSTM's 80 one-byte characters travel as 20 four-byte words
  if (pop->feature_dim != (c->L.model == FL_MODEL_CHAR_LSTM ? 4 * c->L.D_in : c->L.D_in) ||
      (c->L.model == FL_MODEL_CHAR_LSTM && cfg->batch_size != 4)) {
    delete c;
    return FL_ERR_INVALID;
  }
  c->n_pop = pop->n_clients;
  c->n_samples.assign(pop->n_samples, pop->n_samples + pop->n_clients);
  c->pop_off.assign((size_t)c->n_pop + 1, 0);
  for (int64_t k = 0; k < c->n_pop; ++k) {
    if (c->n_samples[(size_t)k] < 0) {
      delete c;
      return FL_ERR_INVALID;
    }
    c->pop_off[(size_t)k + 1] = c->pop_off[(size_t)k] + c->n_samples[(size_t)k];
  }
  c->x = pop->x;
  c->y = pop->y;
  c->pop_dev = pop->on_device != 0;
  *out = c;  // from here on errors are reported through the ctx

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(c, FL_ERR_CUDA, "no CUDA device: this library has no CPU path");
  CK(cudaSetDevice(cfg->device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, cfg->device));
  if (prop.major != 10) return set_err(c, FL_ERR_CUDA, "device %s is sm_%d%d; this build targets sm_100a", prop.name,
                                       prop.major, prop.minor);
  c->n_sms = prop.multiProcessorCount;
  if (cfg->sm_count != 0) {
    std::string why;
    if (!green_partition(cfg->device, cfg->sm_count, &c->green, &why))
      return set_err(c, FL_ERR_CUDA, "sm_count %d: %s", cfg->sm_count, why.c_str());
    c->n_sms = c->green.sms;
  }
  // every stream of the ctx lives in its SM partition (a green-context stream) when one is set
  auto make_stream = [&](cudaStream_t* s, int prio) -> cudaError_t {
    if (c->green.g)
      return c->green.stream_create((CUstream*)s, c->green.g, CU_STREAM_NON_BLOCKING, prio) == CUDA_SUCCESS
                 ? cudaSuccess
                 : cudaErrorInvalidResourceHandle;
    return cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, prio);
  };
  c->solo_sms = c->n_sms;
  if (cfg->stream) c->st = (cudaStream_t)cfg->stream;
  else {
    CK(make_stream(&c->st, 0));
    c->own_stream = true;
  }
  cudaEvent_t* evs[] = {&c->ev_entry, &c->ev_start, &c->ev_staged, &c->ev_trained, &c->ev_agg0,
                        &c->ev_acc1, &c->ev_ar0, &c->ev_ar1, &c->ev_end, &c->ev_tab[0], &c->ev_tab[1]};
  for (cudaEvent_t* e : evs) CK(cudaEventCreate(e));
  for (cudaEvent_t& e : c->ev_sfree) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (const char* ng = getenv("FL_GROUPS")) c->ngroups = std::max(1, atoi(ng));
  if (const char* ns = getenv("FL_SOLO")) c->nsolo = std::max(0, atoi(ns));
  if (const char* ss = getenv("FL_SOLO_SMS")) c->solo_sms = std::max(8, std::min(c->n_sms, atoi(ss)));
  if (const char* rs = getenv("FL_RESERVE_SMS")) c->reserve_sms = std::max(0, std::min(120, atoi(rs)));
  c->reserve_sms = c->reserve_sms * c->n_sms / 148;  // the same share of a smaller partition
  c->nsolo = std::min(c->nsolo, std::max(0, 8 - c->ngroups));
  CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  const int nstreams = c->nsolo + c->ngroups;
  c->gstream.assign((size_t)nstreams, nullptr);
  c->ev_join.assign((size_t)nstreams, nullptr);
  int prio_lo = 0, prio_hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  for (int g = 0; g < nstreams; ++g) {
    const bool hi = g < c->nsolo;  // the critical-path (solo) streams run at high priority
    CK(make_stream(&c->gstream[(size_t)g], hi ? prio_hi : prio_lo));
    CK(cudaEventCreateWithFlags(&c->ev_join[(size_t)g], cudaEventDisableTiming));
  }
  if (!c->pop_dev) {
    CK(make_stream(&c->cst, 0));
    CK(make_stream(&c->pst, prio_hi));
    // borrowed host population: pin it so per-round staging copies run at full PCIe rate
    size_t xb = (size_t)c->pop_off.back() * (size_t)c->L.D_in * sizeof(float);
    if (cudaHostRegister((void*)c->x, xb, cudaHostRegisterReadOnly) == cudaSuccess) c->host_registered = true;
    else cudaGetLastError();
  }
  const int64_t P = c->L.P, Pp = c->L.P_pad;
  CK(cudaMalloc(&c->d_theta, sizeof(float) * Pp));
  CK(cudaMalloc(&c->d_canon_of, sizeof(int64_t) * Pp));
  CK(cudaMalloc(&c->d_canon, sizeof(float) * P));
  CK(cudaMalloc(&c->d_S, sizeof(double) * (Pp + 1)));
  CK(cudaMallocHost(&c->h_rstat, sizeof(double) * 2 * cfg->world_size));
  CK(cudaMalloc(&c->d_rstat, sizeof(double) * (2 + 2 * cfg->world_size)));
  c->peer_T = (int)((Pp + kPeerTile - 1) / kPeerTile);
  CK(cudaMalloc(&c->d_sig, sizeof(unsigned long long) * (FL_MAX_PEERS + 1) * c->peer_T));
  CK(cudaMemset(c->d_sig, 0, sizeof(unsigned long long) * (FL_MAX_PEERS + 1) * c->peer_T));
  CK(cudaMalloc(&c->d_ctr, sizeof(unsigned int) * 2));
  CK(cudaMemset(c->d_ctr, 0, sizeof(unsigned int) * 2));
  CK(cudaMemcpyAsync(c->d_canon_of, c->L.canon_of.data(), sizeof(int64_t) * Pp, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->d_canon, global_params, sizeof(float) * P, cudaMemcpyHostToDevice, c->st));
  canon_to_internal(c->d_canon, c->d_canon_of, Pp, c->d_theta, c->st);
  CKL();
  CK(cudaStreamSynchronize(c->st));
  // a communicator whenever a unique id is given: world_size > 1, or world_size == 1 to run
  // the multi-rank aggregation path (partial -> allreduce -> finalize) on one GPU
  if (cfg->nccl_unique_id) {
    if (!g_nccl.load()) return set_err(c, FL_ERR_NCCL, "cannot dlopen libnccl.so.2");
    ncclUniqueId id;
    memcpy(id.internal, cfg->nccl_unique_id, 128);
    ncclResult_t r = g_nccl.commInitRank(&c->comm, cfg->world_size, id, cfg->rank);
    if (r != ncclSuccess)
      return set_err(c, FL_ERR_NCCL, "ncclCommInitRank: %s", g_nccl.errStr ? g_nccl.errStr(r) : "?");
    int nranks = -1, ver = 0;
    if (g_nccl.commCount) g_nccl.commCount(c->comm, &nranks);
    if (g_nccl.getVersion) g_nccl.getVersion(&ver);
    fprintf(stderr, "[fl] NCCL %d comm ready: rank %d of %d (comm nranks %d) on device %d (%s)\n", ver,
            cfg->rank, cfg->world_size, nranks, cfg->device, prop.name);
    if (nranks != cfg->world_size)
      return set_err(c, FL_ERR_NCCL, "communicator has %d ranks, expected %d", nranks, cfg->world_size);
  }
  return FL_OK;
}

fl_status fl_place(fl_ctx* c, const int64_t* cohort_ids, int64_t n_cohort, int32_t policy, const double* lb_coef,
                   int64_t* out_ids, int64_t* out_off) {
  if (!c) return FL_ERR_INVALID;
  if (c->failed) return FL_ERR_STATE;
  auto t0 = std::chrono::steady_clock::now();
  if (n_cohort < 0 || (n_cohort > 0 && !cohort_ids)) return set_err(c, FL_ERR_INVALID, "bad cohort");
  for (int64_t i = 0; i < n_cohort; ++i) {
    int64_t id = cohort_ids[i];
    if (id >= 0 && id < c->n_pop && c->n_samples[(size_t)id] < c->cfg.min_samples)
      return set_err(c, FL_ERR_INVALID, "client %lld has %lld < min_samples samples", (long long)id,
                     (long long)c->n_samples[(size_t)id]);
  }
  std::vector<int64_t> ids((size_t)n_cohort), off((size_t)c->cfg.world_size + 1);
  int rc = place(policy, cohort_ids, n_cohort, c->n_samples.data(), c->n_pop, c->cfg.batch_size, c->cfg.world_size,
                 lb_coef, ids.data(), off.data());
  if (rc != FL_OK) return set_err(c, (fl_status)rc, "invalid cohort / policy (unknown or duplicate id?)");
  c->plan_ids.swap(ids);
  c->plan_off.swap(off);
  const int r = c->cfg.rank;
  c->local_ids.assign(c->plan_ids.begin() + c->plan_off[(size_t)r], c->plan_ids.begin() + c->plan_off[(size_t)r + 1]);
  c->K_total = n_cohort;
  c->N_total = 0;
  for (int64_t i = 0; i < n_cohort; ++i) c->N_total += c->n_samples[(size_t)cohort_ids[i]];
  c->have_plan = true;
  c->trained = false;
  c->rec_valid = false;  // records describe the previous plan's clients
  if (out_ids) std::copy(c->plan_ids.begin(), c->plan_ids.end(), out_ids);
  if (out_off) std::copy(c->plan_off.begin(), c->plan_off.end(), out_off);
  c->place_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return FL_OK;
}

// Per-round host tables (pinned) -> device, then staging and the SGD waves.
fl_status fl_train_clients(fl_ctx* c, int32_t round_index) {
  if (!c) return FL_ERR_INVALID;
  if (c->failed || !c->have_plan) return set_err(c, FL_ERR_STATE, c->failed ? "ctx failed" : "no plan: call fl_place first");
  CK(cudaSetDevice(c->cfg.device));
  auto t0 = std::chrono::steady_clock::now();
  const Layout& L = c->L;
  const int64_t B = c->cfg.batch_size, E = c->cfg.local_epochs, K = (int64_t)c->local_ids.size();
  // execution order: steps descending (= batches descending), plan order on ties
  c->exec.resize((size_t)K);
  std::iota(c->exec.begin(), c->exec.end(), 0);
  auto nb = [&](int64_t i) { return (c->n_samples[(size_t)c->local_ids[(size_t)i]] + B - 1) / B; };
  // Slot pitch: rows reserved per active client in a wave's activation buffers.  The CNN
  // tensor-core kernels take a client's batch as 32 MMA rows, so a smaller batch (the speech
  // model's B = 20) rides in 32-row slots whose rows >= |b| are padding (sidx = -1).
  const bool cnn_tc = (L.model == FL_MODEL_CNN_CIFAR || L.model == FL_MODEL_CNN_SPEECH) && c->cfg.math == 0;
  const int64_t Bp = (cnn_tc && B < 32) ? 32 : B;
  std::stable_sort(c->exec.begin(), c->exec.end(), [&](int64_t a, int64_t b) { return nb(a) > nb(b); });
  // Groups = concurrent streams. The NS longest clients (the round's critical path) each get
  // a group of their own on a high-priority stream; the rest of the longest-first order is
  // dealt round-robin into NR groups. Each group is contiguous in execution order and itself
  // longest-first, so its active set in every wave is a prefix.
  // Solo groups pay off only when the longest client is a sizeable share of the round's work
  // (its lone-client step latency then sets the round time, e.g. C2: 63 of 819 batches); for a
  // throughput-bound cohort (C3: 63 of 7,951) their reserved SMs and extra streams cost more
  // than they save (measured C3 212.3 -> 207.8 ms without them, C2 13.8 -> 15.3 ms).
  const bool cnn_model = (L.model == FL_MODEL_CNN_CIFAR || L.model == FL_MODEL_CNN_SPEECH);
  int64_t nb_sum = 0;
  for (int64_t i = 0; i < K; ++i) nb_sum += nb(i);
  const bool solo_pays = K > 0 && nb(c->exec[0]) * 32 >= nb_sum;
  const int NS = (cnn_model && solo_pays) ? (int)std::min<int64_t>(c->nsolo, std::max<int64_t>(0, K - 1)) : 0;
  const int NR = cnn_model ? (int)std::max<int64_t>(1, std::min<int64_t>(c->ngroups, K - NS)) : 1;
  const int NG = NS + NR;
  std::vector<int64_t> gsize((size_t)NG, 0);
  {
    std::vector<int64_t> ex2;
    ex2.reserve((size_t)K);
    for (int g = 0; g < NS; ++g) ex2.push_back(c->exec[(size_t)g]), gsize[(size_t)g] = 1;
    for (int r = 0; r < NR; ++r)
      for (int64_t e = NS + r; e < K; e += NR) ex2.push_back(c->exec[(size_t)e]), ++gsize[(size_t)(NS + r)];
    c->exec.swap(ex2);
  }
  c->exec_ids.resize((size_t)K);
  for (int64_t e = 0; e < K; ++e) c->exec_ids[(size_t)e] = c->local_ids[(size_t)c->exec[(size_t)e]];
  c->steps_exec.resize((size_t)K);
  c->n_exec.resize((size_t)K);
  c->pseg.assign((size_t)K + 1, 0);
  c->N_local = 0;
  for (int64_t e = 0; e < K; ++e) {
    int64_t id = c->local_ids[(size_t)c->exec[(size_t)e]];
    c->n_exec[(size_t)e] = c->n_samples[(size_t)id];
    c->steps_exec[(size_t)e] = E * nb(c->exec[(size_t)e]);
    c->pseg[(size_t)e + 1] = c->pseg[(size_t)e] + c->n_exec[(size_t)e];
    c->N_local += c->n_exec[(size_t)e];
  }
  const int64_t R = c->pseg[(size_t)K];
  // Packed row order (every kernel reaches a sample through the per-wave sidx tables, so any
  // order works): chunk-major, client-major inside a chunk.  Chunk q holds batches
  // [chunk_t0[q], chunk_t0[q+1]) of every client — the rows first needed by local SGD step
  // t in that range — so a host population can be staged chunk by chunk while earlier
  // steps train.  Chunks double in length (1, 1, 2, 4, ...); one chunk when the order of
  // a client's rows is shuffled (any step may need any row) or the data is device-resident.
  const bool cnn_pipe = (L.model == FL_MODEL_CNN_CIFAR || L.model == FL_MODEL_CNN_SPEECH) && !c->pop_dev &&
                        !c->cfg.shuffle && getenv("FL_NO_PIPE_STAGE") == nullptr;
  std::vector<int64_t> chunk_t0{0};
  {
    int64_t mmax = 0;
    for (int64_t e = 0; e < K; ++e) mmax = std::max(mmax, (c->n_exec[(size_t)e] + B - 1) / B);
    if (cnn_pipe)
      for (int64_t t = 1; t < mmax; t *= 2) chunk_t0.push_back(t);
    chunk_t0.push_back(std::max<int64_t>(mmax, 1) + (cnn_pipe ? 0 : 1 << 30));
  }
  const int64_t NQ = (int64_t)chunk_t0.size() - 1;
  std::vector<int64_t> cbase((size_t)(K * NQ)), qoff((size_t)NQ + 1, 0);  // cbase[e*NQ+q]: first packed row
  for (int64_t q = 0, r = 0; q < NQ; ++q) {
    qoff[(size_t)q] = r;
    for (int64_t e = 0; e < K; ++e) {
      cbase[(size_t)(e * NQ + q)] = r;
      const int64_t n = c->n_exec[(size_t)e];
      r += std::max<int64_t>(0, std::min(n, chunk_t0[(size_t)q + 1] * B) - std::min(n, chunk_t0[(size_t)q] * B));
    }
    qoff[(size_t)q + 1] = r;
  }
  auto prow = [&](int64_t e, int64_t i) {  // packed row of client e's row i
    const int64_t j = i / B;
    int64_t q = 0;
    while (chunk_t0[(size_t)q + 1] <= j) ++q;
    return cbase[(size_t)(e * NQ + q)] + (i - std::min(i, chunk_t0[(size_t)q] * B));
  };
  WaveSched& ws = c->ws;
  ws.ngroups = NG;
  ws.gbase.assign((size_t)NG + 1, 0);
  ws.gn.assign((size_t)NG, 0);
  ws.gw0.assign((size_t)NG + 1, 0);
  ws.gnw.assign((size_t)NG, 0);
  ws.A.clear();
  ws.slot_off.assign(1, 0);
  ws.bs_off.assign(1, 0);
  ws.gstream.assign((size_t)NG, 0);
  ws.gsolo.assign((size_t)NG, 0);
  for (int g = 0; g < NG; ++g) {
    const int64_t n_g = gsize[(size_t)g];
    ws.gn[(size_t)g] = n_g;
    ws.gstream[(size_t)g] = g < NS ? g : c->nsolo + (g - NS);
    ws.gsolo[(size_t)g] = (g < NS || NS == 0) ? 1 : 0;
    ws.gbase[(size_t)g + 1] = ws.gbase[(size_t)g] + n_g;
    const int64_t b0 = ws.gbase[(size_t)g];
    const int64_t nw = n_g ? c->steps_exec[(size_t)b0] : 0;
    ws.gnw[(size_t)g] = nw;
    ws.gw0[(size_t)g + 1] = ws.gw0[(size_t)g] + nw;
    for (int64_t t = 0; t < nw; ++t) {
      int32_t A = 0;
      while (A < n_g && c->steps_exec[(size_t)(b0 + A)] > t) ++A;  // prefix property within the group
      ws.A.push_back(A);
      ws.slot_off.push_back(ws.slot_off.back() + (int64_t)A * Bp);
      ws.bs_off.push_back(ws.bs_off.back() + A);
    }
  }
  ws.n_waves = (int64_t)ws.A.size();
  const int64_t n_sidx = ws.slot_off[(size_t)ws.n_waves], n_bs = ws.bs_off[(size_t)ws.n_waves];
  // pinned table layout: src_row[R] i64 | n[K] i64 | slot_off[W+1] i64 | sidx i32 | bs i32 | steps[K] i32
  size_t need = sizeof(int64_t) * (size_t)(R + K + ws.n_waves + 1) +
                sizeof(int32_t) * (size_t)(n_sidx + n_bs + K + n_bs + ws.n_waves) + 64;
  const int ti = c->tab_i;
  c->tab_i ^= 1;
  c->tab_wait_ms = 0.0;
  if (c->tab_pending[ti]) {  // round r - 2's table copies (normally long done): not placement time
    auto w0 = std::chrono::steady_clock::now();
    CK(cudaEventSynchronize(c->ev_tab[ti]));
    c->tab_pending[ti] = false;
    c->tab_wait_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
  }
  if (need > c->h_tab_cap[ti]) {
    if (c->h_tab[ti]) cudaFreeHost(c->h_tab[ti]);
    c->h_tab[ti] = nullptr;
    CK(cudaMallocHost(&c->h_tab[ti], need * 2));
    c->h_tab_cap[ti] = need * 2;
  }
  int64_t* h_src = (int64_t*)c->h_tab[ti];
  int64_t* h_n = h_src + R;
  int64_t* h_soff = h_n + K;
  int32_t* h_sidx = (int32_t*)(h_soff + ws.n_waves + 1);
  int32_t* h_bs = h_sidx + n_sidx;
  int32_t* h_steps = h_bs + n_bs;
  int32_t* h_bpre = h_steps + K;  // per wave: prefix sums of |b| over its A clients (A + 1 entries)
  for (int64_t e = 0; e < K; ++e) {
    int64_t id = c->local_ids[(size_t)c->exec[(size_t)e]];
    for (int64_t i = 0; i < c->n_exec[(size_t)e]; ++i) h_src[prow(e, i)] = c->pop_off[(size_t)id] + i;
    h_n[e] = c->n_exec[(size_t)e];
    h_steps[e] = (int32_t)c->steps_exec[(size_t)e];
  }
  for (int64_t t = 0; t <= ws.n_waves; ++t) h_soff[t] = ws.slot_off[(size_t)t];
  // batches: epoch ep of client e uses permutation π_{e,ep} (A5) sliced into m_e batches
  std::vector<int32_t> perm;
  for (int g = 0; g < NG; ++g) {
    for (int64_t el = 0; el < ws.gn[(size_t)g]; ++el) {
      const int64_t e = ws.gbase[(size_t)g] + el;
      const int64_t n = c->n_exec[(size_t)e], m = (n + B - 1) / B;
      const int64_t id = c->local_ids[(size_t)c->exec[(size_t)e]];
      perm.resize((size_t)n);
      for (int64_t ep = 0; ep < E; ++ep) {
        if (c->cfg.shuffle) shuffle_perm(c->cfg.seed, (uint64_t)round_index, (uint64_t)id, (uint64_t)ep, n, perm.data());
        else std::iota(perm.begin(), perm.end(), 0);
        for (int64_t j = 0; j < m; ++j) {
          const int64_t k = ws.gw0[(size_t)g] + ep * m + j;  // flat wave of this step
          int32_t* srow = h_sidx + ws.slot_off[(size_t)k] + el * Bp;
          int32_t bsz = 0;
          for (int64_t r = 0; r < Bp; ++r) {
            const int64_t i = j * B + r;
            if (r < B && i < n) {
              srow[r] = (int32_t)prow(e, perm[(size_t)i]);
              ++bsz;
            } else {
              srow[r] = -1;
            }
          }
          h_bs[ws.bs_off[(size_t)k] + el] = bsz;
        }
      }
    }
  }
  for (int64_t k = 0; k < ws.n_waves; ++k) {
    int32_t* pre = h_bpre + ws.bs_off[(size_t)k] + k;
    pre[0] = 0;
    for (int32_t a = 0; a < ws.A[(size_t)k]; ++a) pre[a + 1] = pre[a] + h_bs[ws.bs_off[(size_t)k] + a];
  }
  // device capacity (grow-only; allocation happens on the first round of a given size)
  CK(grow_dev(c->grave, c->d_slots, c->slots_cap, std::max<int64_t>(K, 1) * L.P_pad));
  CK(grow_dev(c->grave, c->d_xpack, c->xpack_cap, std::max<int64_t>(R, 1) * L.D_pack));
  // shifted planar copies of the input exist only for the tensor-core conv1 dW
  const bool want_planar = L.model == FL_MODEL_CNN_CIFAR && c->cfg.math == 0 && conv1_tc_supported(L);
  if (want_planar)
    CK(grow_dev(c->grave, c->cb.xg, c->cb.xg_cap, (c->xpack_cap / L.D_pack) * conv1_xg_floats()));
  CK(grow_dev(c->grave, c->d_ypack, c->ypack_cap, R));
  CK(grow_dev(c->grave, c->d_src_row, c->src_cap, R));
  CK(grow_dev(c->grave, c->d_n, c->n_cap, K));
  CK(grow_dev(c->grave, c->d_steps, c->steps_cap, K));
  CK(grow_dev(c->grave, c->d_slot_off, c->slot_off_cap, ws.n_waves + 1));
  CK(grow_dev(c->grave, ws.d_sidx, c->sidx_cap, n_sidx));
  CK(grow_dev(c->grave, ws.d_bs, c->bs_cap, n_bs));
  CK(grow_dev(c->grave, ws.d_bpre, c->bpre_cap, n_bs + ws.n_waves));
  if (!c->pop_dev) {
    const int b = c->stage_par;
    CK(grow_dev(c->grave, c->d_stage2[b], c->stage_cap2[b], std::max<int64_t>(R, 1) * L.D_in));
    CK(grow_dev(c->grave, c->d_ystage2[b], c->ystage_cap2[b], R));
    c->d_stage = c->d_stage2[b];
    c->d_ystage = c->d_ystage2[b];
  }
  const bool cnn = (L.model == FL_MODEL_CNN_CIFAR || L.model == FL_MODEL_CNN_SPEECH);
  const bool lstm = L.model == FL_MODEL_CHAR_LSTM;
  if (lstm && K * B > c->lb.slots) {  // wave 0 has every local client active
    LstmBufs& b = c->lb;
    float** bufs[] = {&b.xp, &b.G0, &b.G1, &b.dpre, &b.C0, &b.C1, &b.H0, &b.H1, &b.dX, &b.E, &b.dE, &b.dhT};
    const int kind[] = {0, 0, 0, 0, 1, 1, 1, 1, 2, 3, 3, 4};
    for (int i = 0; i < 12; ++i) {
      if (*bufs[i]) c->grave.push_back(*bufs[i]);  // freed at destroy (see grow_dev)
      *bufs[i] = nullptr;
      CK(cudaMalloc(bufs[i], sizeof(float) * lstm_act_floats(K * B, kind[i])));
    }
    b.slots = K * B;
  }
  if (cnn && K > 0) {
    CnnBufs& b = c->cb;
    const CnnDims& d = L.d;
    b.nch = (int)std::min<int64_t>(8, Bp);
    const int64_t S = (int64_t)K * Bp;  // wave 0 has every local client active
    if (S > c->cb_slots_cap) {
      void* old[] = {b.a1, b.p1, b.a2, b.p2, b.h, b.dh, b.am1, b.am2, b.dp2, b.dY2, b.dp1, b.dY1, b.dz};
      for (void* p : old)
        if (p) c->grave.push_back(p);  // freed at destroy (see grow_dev)
      const int64_t hw0 = (int64_t)d.H0 * d.W0, hw1 = (int64_t)d.H1 * d.W1, hw2 = (int64_t)d.H2 * d.W2;
      // the full-resolution conv1 planes (pre-pool activation, its gradient) exist only on the
      // FP32 SIMT path: the tensor-core / fused paths pool in conv1's epilogue and take conv1's
      // dW from the pooled gradient (4.2 GB each at C3 on one GPU)
      b.a1 = b.dY1 = nullptr;
      if (c->cfg.math != 0) {
        CK(cudaMalloc(&b.a1, sizeof(float) * S * hw0 * d.C1));
        CK(cudaMalloc(&b.dY1, sizeof(float) * S * hw0 * d.C1));
      }
      CK(cudaMalloc(&b.p1, sizeof(float) * S * hw1 * d.C1));
      CK(cudaMalloc(&b.am1, S * hw1 * d.C1));
      CK(cudaMalloc(&b.dp1, sizeof(float) * S * hw1 * d.C1));
      CK(cudaMalloc(&b.a2, sizeof(float) * S * hw1 * d.C2));
      CK(cudaMalloc(&b.dY2, sizeof(float) * S * hw1 * d.C2));
      CK(cudaMalloc(&b.p2, sizeof(float) * S * hw2 * d.C2));
      CK(cudaMalloc(&b.am2, S * hw2 * d.C2));
      CK(cudaMalloc(&b.dp2, sizeof(float) * S * hw2 * d.C2));
      CK(cudaMalloc(&b.h, sizeof(float) * S * d.HID));
      CK(cudaMalloc(&b.dh, sizeof(float) * S * d.HID));
      CK(cudaMalloc(&b.dz, sizeof(float) * S * d.NCLS));
      // batch-padded tensor-core GEMMs read (and multiply by zero) rows past |b|: keep them finite
      CK(cudaMemsetAsync(b.p2, 0, sizeof(float) * S * hw2 * d.C2, c->st));
      CK(cudaMemsetAsync(b.dh, 0, sizeof(float) * S * d.HID, c->st));
      CK(cudaMemsetAsync(b.p1, 0, sizeof(float) * S * hw1 * d.C1, c->st));
      CK(cudaMemsetAsync(b.dY2, 0, sizeof(float) * S * hw1 * d.C2, c->st));
      if (b.dY1) CK(cudaMemsetAsync(b.dY1, 0, sizeof(float) * S * hw0 * d.C1, c->st));
      c->cb_slots_cap = S;
      b.slots = S;
    }
    // split-K partials: one region per group, each holding the larger of the SIMT path's
    // K_g·nch chunks and the tensor-core path's K_g + 2·148 chunks
    const int64_t kg = *std::max_element(gsize.begin(), gsize.end());
    const int64_t pg = std::max<int64_t>(kg * b.nch, conv2_dw_tc_part_z(kg));
    if (pg * NG > c->cb_part_cap) {
      void* old[] = {b.part1, b.part2, b.fc1_part};
      for (void* p : old)
        if (p) c->grave.push_back(p);  // freed at destroy (see grow_dev)
      CK(cudaMalloc(&b.part2, sizeof(float) * NG * pg * std::max<int64_t>(d.C2 * (25 * d.C1 + 1), conv2_dw_tc_z_floats())));
      CK(cudaMalloc(&b.part1, sizeof(float) * NG * pg * d.C1 * (25 * d.cpad + 1)));
      b.fc1_part_floats = (int64_t)160 * 32 * d.HID;
      CK(cudaMalloc(&b.fc1_part, sizeof(float) * NG * b.fc1_part_floats));
      c->cb_part_cap = pg * NG;
    }
    c->part_group_z = pg;
  }
  c->place_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() -
                 c->tab_wait_ms;

  // ---- device work, stream-ordered
  cudaStream_t st = c->st;
  int64_t launches = 0, h2d = 0;
  c->prof.reset();
  CK(cudaEventRecord(c->ev_start, st));
  CK(cudaMemcpyAsync(c->d_src_row, h_src, sizeof(int64_t) * R, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->d_n, h_n, sizeof(int64_t) * K, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->d_slot_off, h_soff, sizeof(int64_t) * (ws.n_waves + 1), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ws.d_sidx, h_sidx, sizeof(int32_t) * n_sidx, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ws.d_bs, h_bs, sizeof(int32_t) * n_bs, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->d_steps, h_steps, sizeof(int32_t) * K, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ws.d_bpre, h_bpre, sizeof(int32_t) * (n_bs + ws.n_waves), cudaMemcpyHostToDevice, st));
  CK(cudaEventRecord(c->ev_tab[ti], st));
  c->tab_pending[ti] = true;
  h2d += (int64_t)(sizeof(int64_t) * (R + K + ws.n_waves + 1) + sizeof(int32_t) * (n_sidx + 2 * n_bs + K + ws.n_waves));
  // stage the cohort's samples: device population -> gather; host population -> H2D copies,
  // chunk by chunk on the copy stream (the previous round has released xpack once st reaches
  // ev_start), each chunk packed as soon as it lands
  const float* xsrc = (const float*)c->x;
  const int32_t* ysrc = c->y;
  const int64_t* srow = c->d_src_row;
  c->prof.begin(st);
  cudaStream_t cs_stage = st;
  int64_t q_issued = 0;
  // With several chunks (pipelined CNN staging) each chunk is staged group by group (exec
  // order is group-contiguous, so a group's rows of a chunk are contiguous) and completes on
  // its own event ev_chunk[q·NGc + g]: a group's waves wait only for their own rows.
  const int64_t NGc = NQ > 1 ? ws.ngroups : 1;
  auto stage_chunk = [&](int64_t q) -> bool {  // H2D of chunk q's rows, then pack them, on cs_stage
    for (int64_t g = 0; g < NGc; ++g) {
      const int64_t e0 = NGc == 1 ? 0 : ws.gbase[(size_t)g], e1 = NGc == 1 ? K : ws.gbase[(size_t)g + 1];
      for (int64_t e = e0; e < e1; ++e) {
        const int64_t n = c->n_exec[(size_t)e];
        const int64_t i0 = std::min(n, chunk_t0[(size_t)q] * B), i1 = std::min(n, chunk_t0[(size_t)q + 1] * B);
        if (i1 <= i0) continue;
        const int64_t id = c->local_ids[(size_t)c->exec[(size_t)e]], r0 = c->pop_off[(size_t)id] + i0;
        const int64_t dst = cbase[(size_t)(e * NQ + q)];
        if (cudaMemcpyAsync(c->d_stage + dst * L.D_in, (const float*)c->x + r0 * L.D_in,
                            sizeof(float) * (i1 - i0) * L.D_in, cudaMemcpyHostToDevice, cs_stage) != cudaSuccess ||
            cudaMemcpyAsync(c->d_ystage + dst, c->y + r0, sizeof(int32_t) * (i1 - i0), cudaMemcpyHostToDevice,
                            cs_stage) != cudaSuccess)
          return false;
      }
      const int64_t q0 = e0 < K ? cbase[(size_t)(e0 * NQ + q)] : qoff[(size_t)q + 1];
      const int64_t nq = (e1 < K ? cbase[(size_t)(e1 * NQ + q)] : qoff[(size_t)q + 1]) - q0;
      // copies stay on the copy stream; the pack of these rows runs on ps once they landed
      cudaStream_t ps = cs_stage == st ? st : c->pst;
      if (ps != cs_stage && (cudaEventRecord(c->ev_copy[(size_t)(q * NGc + g)], cs_stage) != cudaSuccess ||
                             cudaStreamWaitEvent(ps, c->ev_copy[(size_t)(q * NGc + g)], 0) != cudaSuccess))
        return false;
      if (nq > 0) {
        if (cnn)
          launches += pack_cnn(L, c->d_stage + q0 * L.D_in, nullptr, nq, c->d_xpack + q0 * L.D_pack,
                               want_planar ? c->cb.xg + q0 * conv1_xg_floats() : nullptr, ps);
        else
          launches += gather_rows_f32(c->d_stage + q0 * L.D_in, nullptr, nq, L.D_pack, c->d_xpack + q0 * L.D_pack,
                                      ps);
        launches += gather_i32(c->d_ystage + q0, nullptr, nq, c->d_ypack + q0, ps);
      }
      if (cudaEventRecord(c->ev_chunk[(size_t)(q * NGc + g)], ps) != cudaSuccess) return false;
    }
    return true;
  };
  if (!c->pop_dev && R > 0) {
    while ((int64_t)c->ev_chunk.size() < NQ * NGc) {
      cudaEvent_t e, f;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&f, cudaEventDisableTiming));
      c->ev_chunk.push_back(e);
      c->ev_copy.push_back(f);
    }
    cs_stage = c->prof.on ? st : c->cst;  // a profiled round stays serialised on st
    if (cs_stage != st) {
      // the copies only need this staging buffer back (packed two rounds ago); the packs write
      // xpack / xg / ypack, which the previous round reads until st reaches ev_start
      CK(cudaStreamWaitEvent(cs_stage, c->ev_sfree[c->stage_par], 0));
      CK(cudaStreamWaitEvent(c->pst, c->ev_start, 0));
    }
    // chunks 0 and 1 now; chunk q >= 2 is issued from the wave loop when step chunk_t0[q-1]
    // is issued, so the first waves are not queued behind every copy of the round
    for (; q_issued < std::min<int64_t>(NQ, 2); ++q_issued)
      if (!stage_chunk(q_issued)) return set_err(c, FL_ERR_CUDA, "staging copy failed");
    h2d += R * (int64_t)(L.D_in * sizeof(float) + sizeof(int32_t));
    // one chunk: everything waits for it; several: each group waits for its own rows (wave loop)
    if (NQ == 1) CK(cudaStreamWaitEvent(st, c->ev_chunk[0], 0));
  } else {
    if (cnn) launches += pack_cnn(L, xsrc, srow, R, c->d_xpack, want_planar ? c->cb.xg : nullptr, st);
    else launches += gather_rows_f32(xsrc, srow, R, L.D_pack, c->d_xpack, st);
    launches += gather_i32(ysrc, srow, R, c->d_ypack, st);
  }
  c->prof.end(K_PACK, 0, (double)R * (4.0 * (L.D_in + L.D_pack) + 8.0), st);
  CKL();
  CK(cudaEventRecord(c->ev_staged, st));
  // ---- local SGD
  c->cb.xrows = c->xpack_cap / L.D_pack;
  int64_t tl = 0;
  // LB records: event slot per (group, last wave of some client of that group)
  std::vector<int64_t> rec_slot;  // [n_waves] flat wave -> event index or -1
  c->rec_valid = false;
  if (c->rec_on) {
    rec_slot.assign((size_t)ws.n_waves, -1);
    c->rec_of_exec.assign((size_t)K, -1);
    int64_t nev = 0;
    for (int g = 0; g < ws.ngroups; ++g)
      for (int64_t el = 0; el < ws.gn[(size_t)g]; ++el) {
        const int64_t e = ws.gbase[(size_t)g] + el;
        const int64_t k = (lstm || cnn) ? ws.gw0[(size_t)g] + c->steps_exec[(size_t)e] - 1 : 0;
        if (rec_slot[(size_t)k] < 0) rec_slot[(size_t)k] = nev++;
        c->rec_of_exec[(size_t)e] = rec_slot[(size_t)k];
      }
    while ((int64_t)c->rec_ev.size() < nev) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      c->rec_ev.push_back(e);
    }
  }
  if (K > 0) {
    if (cnn) {
      // groups run concurrently on their own streams, forked from and joined into st. Waves
      // are issued wave-major across groups so every stream has work queued from the start.
      // A profiled round runs the groups serialised on st, so each kernel's event interval is
      // its own duration (bench.py's roofline), not time shared with other streams.
      CK(cudaEventRecord(c->ev_fork, st));
      std::vector<CnnBufs> gv((size_t)ws.ngroups);
      std::vector<cudaStream_t> gst((size_t)ws.ngroups, st);
      int64_t max_w = 0;
      for (int g = 0; g < ws.ngroups; ++g) {
        if (ws.gn[(size_t)g] == 0) continue;
        if (!c->prof.on) {
          gst[(size_t)g] = c->gstream[(size_t)ws.gstream[(size_t)g]];
          CK(cudaStreamWaitEvent(gst[(size_t)g], c->ev_fork, 0));
        }
        gv[(size_t)g] = cnn_group_view(c->cb, L.d, (int)Bp, ws.gbase[(size_t)g], ws.gn[(size_t)g], g, c->part_group_z,
                                       conv2_dw_tc_z_floats(), (int64_t)L.d.C1 * (25 * L.d.cpad + 1));
        max_w = std::max(max_w, ws.gnw[(size_t)g]);
      }
      static const bool hostprof = getenv("FL_HOSTPROF") != nullptr;
      const auto th0 = std::chrono::steady_clock::now();
      int64_t next_q = 0;
      const bool piped = !c->pop_dev && R > 0 && NQ > 1;
      for (int64_t t = 0; t < max_w; ++t) {
        while (q_issued < NQ && !c->pop_dev && R > 0 && chunk_t0[(size_t)q_issued - 1] <= t)
          if (!stage_chunk(q_issued++)) return set_err(c, FL_ERR_CUDA, "staging copy failed");
        if (piped && next_q < NQ && t == chunk_t0[(size_t)next_q]) {  // group g's rows of chunk next_q staged
          for (int g = 0; g < ws.ngroups; ++g)
            if (ws.gn[(size_t)g] && t < ws.gnw[(size_t)g])
              CK(cudaStreamWaitEvent(gst[(size_t)g], c->ev_chunk[(size_t)(next_q * NGc + g)], 0));
          ++next_q;
        }
        for (int g = 0; g < ws.ngroups; ++g) {
          if (ws.gn[(size_t)g] == 0 || t >= ws.gnw[(size_t)g]) continue;
          const int64_t k = ws.gw0[(size_t)g] + t, base = ws.gbase[(size_t)g];
          int64_t sum_bs = 0;
          for (int32_t a = 0; a < ws.A[(size_t)k]; ++a) sum_bs += h_bs[ws.bs_off[(size_t)k] + a];
          WaveArgs wa{ws.A[(size_t)k], (int)Bp, t == 0, ws.d_sidx + ws.slot_off[(size_t)k],
                      ws.d_bs + ws.bs_off[(size_t)k], c->cfg.lr, sum_bs, &c->prof, c->cfg.math == 0,
                      ws.gn[(size_t)g], true, ws.d_bpre + ws.bs_off[(size_t)k] + k,
                      (ws.gsolo[(size_t)g] || c->reserve_sms == 0) ? c->solo_sms : c->n_sms - c->reserve_sms};
          int nl = cnn_wave_simt(L, wa, c->d_xpack, c->d_ypack, c->d_theta, c->d_slots + base * L.P_pad,
                                 gv[(size_t)g], gst[(size_t)g]);
          if (nl < 0)
            return set_err(c, FL_ERR_CUDA, "tensor-core kernel launch / tensor map failed (group %d wave %lld)", g,
                           (long long)t);
          tl += nl;
          if (c->rec_on && rec_slot[(size_t)k] >= 0)
            CK(cudaEventRecord(c->rec_ev[(size_t)rec_slot[(size_t)k]], gst[(size_t)g]));
        }
      }
      if (hostprof)
        fprintf(stderr, "[fl] issued %lld launches for %lld waves in %.3f ms host time\n", (long long)tl,
                (long long)ws.n_waves,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count());
      for (int g = 0; g < ws.ngroups; ++g) {
        if (ws.gn[(size_t)g] == 0 || gst[(size_t)g] == st) continue;
        CK(cudaEventRecord(c->ev_join[(size_t)g], gst[(size_t)g]));
        CK(cudaStreamWaitEvent(st, c->ev_join[(size_t)g], 0));
      }
    } else if (lstm) {
      for (int64_t k = 0; k < ws.n_waves; ++k) {
        int64_t sum_bs = 0;
        for (int32_t a = 0; a < ws.A[(size_t)k]; ++a) sum_bs += h_bs[ws.bs_off[(size_t)k] + a];
        WaveArgs wa{ws.A[(size_t)k], (int)B, k == 0, ws.d_sidx + ws.slot_off[(size_t)k], ws.d_bs + ws.bs_off[(size_t)k],
                    c->cfg.lr, sum_bs, &c->prof, c->cfg.math == 0, K, true, ws.d_bpre + ws.bs_off[(size_t)k] + k, c->n_sms};
        c->prof.begin(st);
        const int nl = lstm_wave(L, wa, reinterpret_cast<const uint8_t*>(c->d_xpack), c->d_ypack, c->d_theta,
                                 c->d_slots, c->lb, st);
        if (nl < 0) return set_err(c, FL_ERR_CUDA, "lstm wave %lld launch failed", (long long)k);
        c->prof.end(K_LSTM, 381.5e6 * (double)sum_bs, 2.0 * 4.0 * ws.A[(size_t)k] * L.P_pad, st);
        tl += nl;
        if (c->rec_on && rec_slot[(size_t)k] >= 0) CK(cudaEventRecord(c->rec_ev[(size_t)rec_slot[(size_t)k]], st));
      }
    } else {
      c->prof.begin(st);
      tl += logreg_train(L, ws, (int)K, (int)B, c->cfg.lr, c->d_xpack, c->d_ypack, c->d_theta, c->d_slots,
                         c->d_steps, c->d_slot_off, st);
      double S = 0;
      for (int64_t e = 0; e < K; ++e) S += (double)c->n_exec[(size_t)e] * E;
      c->prof.end(K_LOGREG, 3.0 * 2.0 * S * 7840, 4.0 * S * 785 + 8.0 * K * L.P_pad, st);
      // one CTA per client inside one launch: every client's record is the launch's end
      if (c->rec_on) CK(cudaEventRecord(c->rec_ev[0], st));
    }
    CKL();
  }
  c->rec_valid = c->rec_on;
  CK(cudaEventRecord(c->ev_trained, st));
  if (!c->pop_dev && R > 0) {  // every chunk of this round was packed on pst: its buffer is free after that
    CK(cudaEventRecord(c->ev_sfree[c->stage_par], c->prof.on ? st : c->pst));
    c->stage_par ^= 1;
  }
  c->kernels = launches + tl;
  c->train_launches = tl;
  c->h2d = h2d;
  c->trained = true;
  return FL_OK;
}

static fl_status aggregate(fl_ctx* c, float* out_params, int64_t* out_total_samples, bool sync);

fl_status fl_aggregate(fl_ctx* c, float* out_params, int64_t* out_total_samples) {
  return aggregate(c, out_params, out_total_samples, true);
}

fl_status fl_aggregate_async(fl_ctx* c, float* out_params, int64_t* out_total_samples) {
  if (!c) return FL_ERR_INVALID;
  if (out_params) {  // an async D2H into pageable memory would silently synchronise the host
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, out_params) != cudaSuccess || at.type != cudaMemoryTypeHost) {
      cudaGetLastError();
      return set_err(c, FL_ERR_INVALID, "fl_aggregate_async: out_params must be page-locked host memory");
    }
  }
  return aggregate(c, out_params, out_total_samples, false);
}

fl_status fl_synchronize(fl_ctx* c) {
  if (!c) return FL_ERR_INVALID;
  CK(cudaSetDevice(c->cfg.device));
  CK(cudaStreamSynchronize(c->st));
  return FL_OK;
}

static fl_status aggregate(fl_ctx* c, float* out_params, int64_t* out_total_samples, bool sync) {
  if (!c) return FL_ERR_INVALID;
  if (c->failed || !c->trained) return set_err(c, FL_ERR_STATE, c->failed ? "ctx failed" : "train before aggregate");
  if (c->N_total <= 0) return set_err(c, FL_ERR_EMPTY, "total sample count is 0");
  CK(cudaSetDevice(c->cfg.device));
  const int64_t Pp = c->L.P_pad, K = (int64_t)c->exec.size();
  cudaStream_t st = c->st;
  CK(cudaEventRecord(c->ev_agg0, st));
  int64_t n = 0;
  c->prof.begin(st);
  const double agg_bytes = 4.0 * (double)Pp * (double)(K + 1) + (c->comm ? 8.0 : 4.0) * (double)Pp;
  const int W = c->cfg.world_size;
  const int mode = c->cfg.agg_mode;
  if (mode != FL_AGG_NCCL && W > 1 && !c->peer_on)
    return set_err(c, FL_ERR_STATE, "agg_mode %d needs fl_peer_connect first", mode);
  c->xfer_bytes = 0;
  if (c->peer_on && mode == FL_AGG_PEER) {
    // one cooperative kernel: partial, reduce-scatter over peer memory, finalize, all-gather
    PeerArgs a = c->peer;
    a.slots = c->d_slots, a.stride = Pp, a.n = c->d_n, a.K = (int)K, a.N = (double)c->N_total;
    a.seq = ++c->agg_seq;
    CK(cudaEventRecord(c->ev_acc1, st));
    CK(cudaEventRecord(c->ev_ar0, st));
    if (fedavg_peer(a, c->n_sms, st) < 0) return set_err(c, FL_ERR_CUDA, "k_fedavg_peer launch failed");
    ++n;
    CKL();
    CK(cudaEventRecord(c->ev_ar1, st));
    c->prof.end(K_FEDAVG, 3.0 * (double)Pp * K, agg_bytes, st);
    const int64_t t0 = peer_slice_begin(a.me, a.T, W), t1 = peer_slice_begin(a.me + 1, a.T, W);
    const int64_t slice = std::min<int64_t>(Pp, t1 * kPeerTile) - std::min<int64_t>(Pp, t0 * kPeerTile);
    c->xfer_bytes = (int64_t)(W - 1) * slice * 12;  // pull 8 B of every peer's S, push 4 B of θ_new
  } else if (c->peer_on && mode == FL_AGG_UNAGGREGATED) {
    // the ablation: every client model to the server (rank 0), which averages all of them
    const int r = c->cfg.rank;
    const int64_t Kt = c->K_total;
    if (c->peer.r[0].recv == nullptr || Kt > c->recv_cap)
      return set_err(c, FL_ERR_INVALID, "unaggregated: server receive buffer holds %lld models, cohort has %lld",
                     (long long)c->recv_cap, (long long)Kt);
    std::vector<int64_t> dst((size_t)K);
    for (int64_t e = 0; e < K; ++e) dst[(size_t)e] = c->plan_off[(size_t)r] + c->exec[(size_t)e];
    CK(grow_dev(c->grave, c->d_dst_row, c->dst_cap, K));
    if (K) CK(cudaMemcpyAsync(c->d_dst_row, dst.data(), sizeof(int64_t) * K, cudaMemcpyHostToDevice, st));
    const unsigned long long seq = ++c->agg_seq;
    CK(cudaEventRecord(c->ev_acc1, st));
    CK(cudaEventRecord(c->ev_ar0, st));
    n += unagg_push(c->d_slots, Pp, c->d_dst_row, (int)K, Pp / 4, c->peer.r[0].recv, c->peer.r[0].sig, r, seq,
                    c->d_ctr, c->n_sms, st);
    if (r != 0) {
      c->xfer_bytes = K * Pp * 4;
      n += wait_flags(c->d_sig + (int64_t)W * c->peer_T, 0, 1, 1, seq, st);  // θ_new from the server
    } else {
      std::vector<int64_t> np((size_t)Kt);
      for (int64_t i = 0; i < Kt; ++i) np[(size_t)i] = c->n_samples[(size_t)c->plan_ids[(size_t)i]];
      CK(grow_dev(c->grave, c->d_nplan, c->nplan_cap, Kt));
      CK(cudaMemcpyAsync(c->d_nplan, np.data(), sizeof(int64_t) * Kt, cudaMemcpyHostToDevice, st));
      n += wait_flags(c->d_sig, 0, W, 1, seq, st);  // every rank's models have landed
      n += fedavg_accum_final(c->d_recv, Pp, c->d_nplan, (int)Kt, Pp, c->d_theta, (double)c->N_total, c->d_theta, st);
      PeerArgs a = c->peer;
      a.seq = seq;
      n += unagg_bcast(a, c->d_ctr + 1, c->n_sms, st);
      c->xfer_bytes = (int64_t)(W - 1) * Pp * 4;
    }
    CKL();
    CK(cudaEventRecord(c->ev_ar1, st));
    c->prof.end(K_FEDAVG, 3.0 * (double)Pp * Kt, 4.0 * (double)Pp * (double)(Kt + 1) + 4.0 * (double)Pp, st);
  } else if (!c->comm) {
    n += fedavg_accum_final(c->d_slots, Pp, c->d_n, (int)K, Pp, c->d_theta, (double)c->N_total, c->d_theta, st);
    CKL();
    c->prof.end(K_FEDAVG, 3.0 * (double)Pp * K, agg_bytes, st);
    CK(cudaEventRecord(c->ev_acc1, st));
    CK(cudaEventRecord(c->ev_ar0, st));
    CK(cudaEventRecord(c->ev_ar1, st));
  } else {
    // [S_g ‖ N_g]: N_g travels as a kernel argument (no pinned host scalar that a queued
    // next round could overwrite before an asynchronous copy reads it)
    n += fedavg_accum_partial(c->d_slots, Pp, c->d_n, (int)K, Pp, c->d_theta, (double)c->N_local, c->d_S, st);
    CKL();
    c->prof.end(K_FEDAVG, 3.0 * (double)Pp * K, agg_bytes, st);
    CK(cudaEventRecord(c->ev_acc1, st));
    CK(cudaEventRecord(c->ev_ar0, st));
    ncclResult_t r = g_nccl.allReduce(c->d_S, c->d_S, (size_t)(Pp + 1), ncclFloat64, ncclSum, c->comm, st);
    if (r != ncclSuccess) return set_err(c, FL_ERR_NCCL, "ncclAllReduce: %s", g_nccl.errStr ? g_nccl.errStr(r) : "?");
    CK(cudaEventRecord(c->ev_ar1, st));
    n += fedavg_finalize(c->d_S, Pp, c->d_theta, c->d_S + Pp, c->d_theta, st);
    CKL();
    c->xfer_bytes = W > 1 ? (int64_t)(2.0 * (W - 1) / W * 8.0 * (double)(Pp + 1)) : 0;  // ring estimate
  }
  CK(cudaEventRecord(c->ev_end, st));
  c->kernels += n;
  c->trained = false;
  c->have_plan = false;
  if (out_total_samples) *out_total_samples = c->N_total;
  if (out_params) {
    internal_to_canon(c->d_theta, c->d_canon_of, Pp, c->d_canon, st);
    CKL();
    CK(cudaMemcpyAsync(out_params, c->d_canon, sizeof(float) * c->L.P, cudaMemcpyDeviceToHost, st));
    if (sync) CK(cudaStreamSynchronize(st));
  }
  return FL_OK;
}

static double ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();
    return 0.0;
  }
  return ms;
}

// Per-rank device times of the last round; with a communicator, [round_ms, train_end_ms] of
// every rank are all-gathered (8·2·world bytes on the ctx stream) for the max-over-ranks round
// time and the "timedelta workers" statistic.  Collective when a
// communicator exists: every rank must call it.
static fl_status fill_stats(fl_ctx* c, fl_round_stats* s) {
  memset(s, 0, sizeof *s);
  s->round_ms = ev_ms(c->ev_entry, c->ev_end);
  s->train_end_ms = ev_ms(c->ev_entry, c->ev_trained);
  s->round_ms_max = s->round_ms;
  s->train_end_ms_min = s->train_end_ms_max = s->train_end_ms;
  if (c->comm) {
    const int W = c->cfg.world_size;
    const double mine[2] = {s->round_ms, s->train_end_ms};
    CK(cudaMemcpyAsync(c->d_rstat, mine, sizeof mine, cudaMemcpyHostToDevice, c->st));  // pageable: staged now
    ncclResult_t r = g_nccl.allGather(c->d_rstat, c->d_rstat + 2, 2, ncclFloat64, c->comm, c->st);
    if (r != ncclSuccess) return set_err(c, FL_ERR_NCCL, "ncclAllGather: %s", g_nccl.errStr ? g_nccl.errStr(r) : "?");
    CK(cudaMemcpyAsync(c->h_rstat, c->d_rstat + 2, sizeof(double) * 2 * W, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    for (int w = 0; w < W; ++w) {
      s->round_ms_max = std::max(s->round_ms_max, c->h_rstat[2 * w]);
      s->train_end_ms_min = std::min(s->train_end_ms_min, c->h_rstat[2 * w + 1]);
      s->train_end_ms_max = std::max(s->train_end_ms_max, c->h_rstat[2 * w + 1]);
    }
  }
  s->timedelta_ms = s->train_end_ms_max - s->train_end_ms_min;
  s->place_ms = c->place_ms;
  s->stage_ms = ev_ms(c->ev_start, c->ev_staged);
  s->train_ms = ev_ms(c->ev_staged, c->ev_trained);
  s->agg_ms = ev_ms(c->ev_agg0, c->ev_end);
  s->allreduce_ms = ev_ms(c->ev_ar0, c->ev_ar1);
  s->clients_total = c->K_total;
  s->clients_local = (int64_t)c->exec.size();
  s->samples_total = c->N_total;
  s->samples_local = c->N_local;
  for (int64_t v : c->steps_exec) s->steps_local += v;
  s->waves = c->ws.n_waves;
  s->h2d_bytes = c->h2d;
  s->kernels = c->kernels;
  s->xfer_bytes = c->xfer_bytes;
  s->sm_count = c->n_sms;
  s->client_updates_per_s = s->round_ms_max > 0 ? (double)c->K_total / (s->round_ms_max * 1e-3) : 0.0;
  return FL_OK;
}

fl_status fl_round(fl_ctx* c, const int64_t* cohort_ids, int64_t n_cohort, int32_t policy, const double* lb_coef,
                   int32_t round_index, fl_round_stats* stats) {
  if (!c) return FL_ERR_INVALID;
  if (c->failed) return set_err(c, FL_ERR_STATE, "ctx failed");
  CK(cudaSetDevice(c->cfg.device));
  CK(cudaEventRecord(c->ev_entry, c->st));
  fl_status s = fl_place(c, cohort_ids, n_cohort, policy, lb_coef, nullptr, nullptr);
  if (s != FL_OK) return s;
  s = fl_train_clients(c, round_index);
  if (s != FL_OK) return s;
  s = fl_aggregate(c, nullptr, nullptr);
  if (s != FL_OK) return s;
  if (stats) {
    CK(cudaEventSynchronize(c->ev_end));
    s = fill_stats(c, &c->stats);
    if (s != FL_OK) return s;
    *stats = c->stats;
  }
  return FL_OK;
}

fl_status fl_peer_export(fl_ctx* c, int64_t max_clients, uint8_t* out_blob) {
  if (!c || !out_blob || max_clients < 0) return FL_ERR_INVALID;
  if (c->failed) return FL_ERR_STATE;
  if (c->cfg.agg_mode == FL_AGG_NCCL) return set_err(c, FL_ERR_INVALID, "agg_mode is NCCL: nothing to export");
  CK(cudaSetDevice(c->cfg.device));
  const int64_t Pp = c->L.P_pad;
  if (c->cfg.agg_mode == FL_AGG_UNAGGREGATED && c->cfg.rank == 0 && max_clients > c->recv_cap) {
    if (c->d_recv) cudaFree(c->d_recv);
    c->d_recv = nullptr;
    c->recv_cap = 0;
    CK(cudaMalloc(&c->d_recv, sizeof(float) * (size_t)(max_clients * Pp)));
    c->recv_cap = max_clients;
  }
  PeerBlob b;
  memset(&b, 0, sizeof b);
  b.magic = kPeerMagic;
  b.pid = (int32_t)getpid();
  b.device = c->cfg.device;
  b.sm_count = c->cfg.sm_count;
  b.world = c->cfg.world_size;
  b.rank = c->cfg.rank;
  b.T = c->peer_T;
  b.P_pad = Pp;
  b.recv_cap = c->recv_cap;
  void* ptrs[4] = {c->d_S, c->d_theta, c->d_sig, c->d_recv};
  for (int i = 0; i < 4; ++i) {
    b.ptr[i] = (uint64_t)(uintptr_t)ptrs[i];
    if (ptrs[i]) CK(cudaIpcGetMemHandle(&b.h[i], ptrs[i]));
  }
  memset(out_blob, 0, FL_PEER_BLOB_BYTES);
  memcpy(out_blob, &b, sizeof b);
  return FL_OK;
}

fl_status fl_peer_connect(fl_ctx* c, const uint8_t* blobs, int32_t world) {
  if (!c || !blobs) return FL_ERR_INVALID;
  if (c->failed) return FL_ERR_STATE;
  if (c->cfg.agg_mode == FL_AGG_NCCL) return set_err(c, FL_ERR_INVALID, "agg_mode is NCCL");
  if (world != c->cfg.world_size) return set_err(c, FL_ERR_INVALID, "%d blobs for world_size %d", world, c->cfg.world_size);
  if (c->peer_on) return set_err(c, FL_ERR_STATE, "already connected");
  std::vector<PeerBlob> b((size_t)world);
  for (int j = 0; j < world; ++j) {
    memcpy(&b[(size_t)j], blobs + (size_t)j * FL_PEER_BLOB_BYTES, sizeof(PeerBlob));
    const PeerBlob& x = b[(size_t)j];
    if (x.magic != kPeerMagic || x.rank != j || x.world != world || x.T != c->peer_T || x.P_pad != c->L.P_pad)
      return set_err(c, FL_ERR_INVALID, "peer blob %d does not match this ctx (rank, world, model)", j);
  }
  const int me = c->cfg.rank, pid = (int)getpid();
  if (b[(size_t)me].pid != pid || b[(size_t)me].ptr[1] != (uint64_t)(uintptr_t)c->d_theta)
    return set_err(c, FL_ERR_INVALID, "blob %d is not this ctx's", me);
  for (int j = 0; j < world; ++j)
    for (int i = j + 1; i < world; ++i)
      if (b[(size_t)j].device == b[(size_t)i].device) {
        // a rank's aggregation kernel waits on the device for its peers: ranks sharing a GPU
        // must run concurrently, i.e. in one process on disjoint SM partitions
        if (b[(size_t)j].pid != b[(size_t)i].pid || b[(size_t)j].sm_count == 0 || b[(size_t)i].sm_count == 0)
          return set_err(c, FL_ERR_INVALID, "ranks %d and %d share device %d: they must be contexts of one process "
                         "with SM partitions (sm_count)", j, i, b[(size_t)j].device);
      }
  CK(cudaSetDevice(c->cfg.device));
  if (peer_preload() != 0) return set_err(c, FL_ERR_CUDA, "cannot load the peer-aggregation kernels");
  PeerArgs a{};
  a.W = world, a.me = me, a.T = c->peer_T, a.P4 = c->L.P_pad / 4, a.tile4 = kPeerTile / 4;
  for (int j = 0; j < world; ++j) {
    const PeerBlob& x = b[(size_t)j];
    void* p[4] = {nullptr, nullptr, nullptr, nullptr};
    if (x.pid == pid) {
      for (int i = 0; i < 4; ++i) p[i] = (void*)(uintptr_t)x.ptr[i];
      if (x.device != c->cfg.device) {
        int can = 0;
        CK(cudaDeviceCanAccessPeer(&can, c->cfg.device, x.device));
        if (!can) return set_err(c, FL_ERR_CUDA, "no peer access from device %d to %d", c->cfg.device, x.device);
        cudaError_t e = cudaDeviceEnablePeerAccess(x.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
        cudaGetLastError();
      }
    } else {
      for (int i = 0; i < 4; ++i) {
        if (!x.ptr[i]) continue;
        if (i == 3 && !(j == 0 && c->cfg.agg_mode == FL_AGG_UNAGGREGATED)) continue;
        CK(cudaIpcOpenMemHandle(&p[i], x.h[i], cudaIpcMemLazyEnablePeerAccess));
        c->ipc_opened.push_back(p[i]);
      }
    }
    a.r[j] = PeerRank{(double*)p[0], (float*)p[1], (unsigned long long*)p[2], (float*)p[3]};
  }
  if (c->cfg.agg_mode == FL_AGG_UNAGGREGATED) {
    if (!a.r[0].recv) return set_err(c, FL_ERR_INVALID, "server (rank 0) exported no receive buffer (max_clients)");
    c->recv_cap = b[0].recv_cap;
  }
  c->peer = a;
  c->peer_on = true;
  return FL_OK;
}

fl_status fl_set_timing_records(fl_ctx* c, int32_t on) {
  if (!c) return FL_ERR_INVALID;
  c->rec_on = on != 0;
  return FL_OK;
}

fl_status fl_get_client_times(fl_ctx* c, int64_t* ids, int64_t* m, double* t_ms, int64_t* n_local) {
  if (!c) return FL_ERR_INVALID;
  if (!c->rec_valid) return set_err(c, FL_ERR_STATE, "no round trained with timing records on");
  const int64_t K = (int64_t)c->exec.size(), B = c->cfg.batch_size;
  if (n_local) *n_local = K;
  if (!ids && !m && !t_ms) return FL_OK;
  CK(cudaSetDevice(c->cfg.device));
  CK(cudaEventSynchronize(c->ev_trained));
  // exec order -> plan order
  for (int64_t e = 0; e < K; ++e) {
    const int64_t i = c->exec[(size_t)e];  // index into local_ids (plan order)
    const int64_t id = c->local_ids[(size_t)i];
    if (ids) ids[i] = id;
    if (m) m[i] = (c->n_samples[(size_t)id] + B - 1) / B;
    if (t_ms) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c->ev_staged, c->rec_ev[(size_t)c->rec_of_exec[(size_t)e]]));
      t_ms[i] = ms;
    }
  }
  return FL_OK;
}

fl_status fl_get_stats(fl_ctx* c, fl_round_stats* out) {
  if (!c || !out) return FL_ERR_INVALID;
  if (c->failed) return FL_ERR_STATE;
  CK(cudaSetDevice(c->cfg.device));
  CK(cudaEventSynchronize(c->ev_end));
  fl_status s = fill_stats(c, &c->stats);
  if (s != FL_OK) return s;
  *out = c->stats;
  return FL_OK;
}

fl_status fl_set_profiling(fl_ctx* c, int32_t on) {
  if (!c) return FL_ERR_INVALID;
  c->prof.on = on != 0;
  return FL_OK;
}

fl_status fl_get_kernel_stats(fl_ctx* c, int32_t kind, fl_kernel_stats* out) {
  if (!c || !out || kind < 0 || kind >= K_NKINDS) return FL_ERR_INVALID;
  CK(cudaSetDevice(c->cfg.device));
  CK(cudaStreamSynchronize(c->st));
  memset(out, 0, sizeof *out);
  snprintf(out->name, sizeof out->name, "%s", kKindName[kind]);
  for (const KRec& r : c->prof.recs) {
    if (r.kind != kind) continue;
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, r.a, r.b));
    out->ms += ms;
    out->launches += 1;
    out->flops += r.flops;
    out->bytes += r.bytes;
  }
  return FL_OK;
}

fl_status fl_fedavg_vectors(fl_ctx* c, const float* theta_k, const int64_t* n, int64_t K, int64_t P,
                            const float* theta_g, float* out) {
  if (!c || !theta_k || !n || !theta_g || !out || K < 1 || P < 1) return FL_ERR_INVALID;
  if (c->failed) return FL_ERR_STATE;
  int64_t N = 0;
  for (int64_t k = 0; k < K; ++k) {
    if (n[k] < 1) return set_err(c, FL_ERR_INVALID, "weight < 1");
    N += n[k];
  }
  CK(cudaSetDevice(c->cfg.device));
  CK(grow_dev(c->grave, c->d_n, c->n_cap, K));
  CK(cudaMemcpyAsync(c->d_n, n, sizeof(int64_t) * K, cudaMemcpyHostToDevice, c->st));
  CK(cudaEventRecord(c->ev_agg0, c->st));
  fedavg_accum_final(theta_k, P, c->d_n, (int)K, P, theta_g, (double)N, out, c->st);
  CKL();
  CK(cudaEventRecord(c->ev_acc1, c->st));
  CK(cudaStreamSynchronize(c->st));
  return FL_OK;
}

fl_status fl_get_local_plan(fl_ctx* c, int64_t* ids, int64_t* seg_off, int64_t* steps, int64_t* n_local) {
  if (!c || !n_local) return FL_ERR_INVALID;
  const int64_t K = (int64_t)c->local_ids.size();
  *n_local = K;
  if (ids) std::copy(c->local_ids.begin(), c->local_ids.end(), ids);
  if (seg_off || steps)
    return (fl_status)pack(c->local_ids.data(), K, c->n_samples.data(), c->n_pop, c->cfg.batch_size,
                           c->cfg.local_epochs, seg_off, steps);
  return FL_OK;
}

fl_status fl_get_client_params(fl_ctx* c, int64_t client_id, float* out) {
  if (!c || !out) return FL_ERR_INVALID;
  if (c->failed) return FL_ERR_STATE;
  int64_t e = -1;  // exec position in the last trained round (fl_place does not change it)
  for (size_t i = 0; i < c->exec_ids.size(); ++i)
    if (c->exec_ids[i] == client_id) e = (int64_t)i;
  if (e < 0 || !c->d_slots) return set_err(c, FL_ERR_INVALID, "client %lld not trained on this rank", (long long)client_id);
  CK(cudaSetDevice(c->cfg.device));
  internal_to_canon(c->d_slots + e * c->L.P_pad, c->d_canon_of, c->L.P_pad, c->d_canon, c->st);
  CKL();
  CK(cudaMemcpyAsync(out, c->d_canon, sizeof(float) * c->L.P, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return FL_OK;
}

fl_status fl_get_global_params(fl_ctx* c, float* out) {
  if (!c || !out) return FL_ERR_INVALID;
  if (c->failed) return FL_ERR_STATE;
  CK(cudaSetDevice(c->cfg.device));
  internal_to_canon(c->d_theta, c->d_canon_of, c->L.P_pad, c->d_canon, c->st);
  CKL();
  CK(cudaMemcpyAsync(out, c->d_canon, sizeof(float) * c->L.P, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return FL_OK;
}

fl_status fl_set_global_params(fl_ctx* c, const float* params) {
  if (!c || !params) return FL_ERR_INVALID;
  if (c->failed) return FL_ERR_STATE;
  CK(cudaSetDevice(c->cfg.device));
  CK(cudaMemcpyAsync(c->d_canon, params, sizeof(float) * c->L.P, cudaMemcpyHostToDevice, c->st));
  canon_to_internal(c->d_canon, c->d_canon_of, c->L.P_pad, c->d_theta, c->st);
  CKL();
  CK(cudaStreamSynchronize(c->st));
  return FL_OK;
}

fl_status fl_debug_read(fl_ctx* c, const char* name, void* host, int64_t bytes) {
  if (!c || !name || !host || bytes < 0) return FL_ERR_INVALID;
  if (strcmp(name, "sig") == 0) {  // peer signal words, read without synchronising the ctx stream
    CK(cudaSetDevice(c->cfg.device));
    CK(cudaMemcpy(host, c->d_sig,
                  (size_t)std::min<int64_t>(bytes, sizeof(unsigned long long) * (FL_MAX_PEERS + 1) * c->peer_T),
                  cudaMemcpyDeviceToHost));
    return FL_OK;
  }
  if (c->L.model != FL_MODEL_CNN_CIFAR && c->L.model != FL_MODEL_CNN_SPEECH) return FL_ERR_INVALID;
  const CnnBufs& b = c->cb;
  const CnnDims& d = c->L.d;
  const int64_t S = b.slots, hw0 = (int64_t)d.H0 * d.W0, hw1 = (int64_t)d.H1 * d.W1, hw2 = (int64_t)d.H2 * d.W2;
  struct { const char* n; const void* p; int64_t bytes; } tab[] = {
      {"p1", b.p1, 4 * S * hw1 * d.C1}, {"am1", b.am1, S * hw1 * d.C1}, {"p2", b.p2, 4 * S * hw2 * d.C2},
      {"am2", b.am2, S * hw2 * d.C2},   {"h", b.h, 4 * S * d.HID},      {"dh", b.dh, 4 * S * d.HID},
      {"dp2", b.dp2, 4 * S * d.F},      {"dY2", b.dY2, 4 * S * hw1 * d.C2}, {"dp1", b.dp1, 4 * S * hw1 * d.C1},
      {"dY1", b.dY1, 4 * S * hw0 * d.C1}};
  for (auto& t : tab) {
    if (strcmp(t.n, name) != 0) continue;
    if (!t.p) return set_err(c, FL_ERR_STATE, "buffer %s not allocated yet", name);
    CK(cudaSetDevice(c->cfg.device));
    CK(cudaStreamSynchronize(c->st));
    CK(cudaMemcpy(host, t.p, (size_t)std::min<int64_t>(bytes, t.bytes), cudaMemcpyDeviceToHost));
    return FL_OK;
  }
  return set_err(c, FL_ERR_INVALID, "unknown buffer %s", name);
}

}  // extern "C"

