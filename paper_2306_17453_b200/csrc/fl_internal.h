// fl_internal.h — internal declarations shared by the library's translation units.
// Nothing here is part of the ABI (see include/fl.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdlib.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/fl.h"

namespace flb {

// Programmatic dependent launch: the kernel may begin while its stream predecessor drains;
// it must call pdl_trigger() / pdl_wait() (dev_util.cuh) before touching any data the
// predecessor produces. FL_PDL=0 turns it off (plain stream order).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("FL_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(bool on, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = (on && pdl_enabled()) ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- model geometry
// CNN family (McMahan CNN on CIFAR / speech, reading A10): conv5x5 'same' + ReLU +
// maxpool2 -> conv5x5 'same' + ReLU + maxpool2 -> fc + ReLU -> fc.
struct CnnDims {
  int cin, cpad;       // input channels, padded to 4 for 16-byte NHWC pixels
  int H0, W0;          // input
  int C1, C2;          // conv channels (32, 64)
  int H1, W1, H2, W2;  // after pool1 / pool2 (floor)
  int F;               // C2*H2*W2 (fc1 fan-in)
  int HID, NCLS;
};

// Internal (device) parameter layout: NHWC-friendly, every tensor 128-byte aligned.
//   c1w [C1][5][5][cpad]  c1b [C1]  c2w [C2][5][5][C1]  c2b [C2]
//   f1w [HID][H2][W2][C2] f1b [HID] f2w [NCLS][HID]     f2b [NCLS]
// logreg: w [10][784] b [10].   LSTM: canonical order (see lstm kernels).
// char-LSTM parameter offsets (canonical torch order, every tensor 128-byte aligned)
struct LstmOff {
  int64_t emb = 0, wih[2] = {0, 0}, whh[2] = {0, 0}, bih[2] = {0, 0}, bhh[2] = {0, 0}, wfc = 0, bfc = 0;
};

struct Layout {
  int model = -1;
  int64_t P = 0;      // canonical parameter count
  int64_t P_pad = 0;  // internal per-slot stride (floats, multiple of 32)
  int D_in = 0;       // population feature dim
  int D_pack = 0;     // packed per-sample floats (NHWC4 for CNN)
  CnnDims d{};
  int64_t o_c1w = 0, o_c1b = 0, o_c2w = 0, o_c2b = 0, o_f1w = 0, o_f1b = 0, o_f2w = 0, o_f2b = 0;
  LstmOff lo;
  std::vector<int64_t> canon_of;  // [P_pad]: canonical index of each internal slot, -1 = padding
};

bool make_layout(int model, Layout* L);

// ---------------------------------------------------------------- per-wave schedule
// Wave t = SGD step t of every local client with more than t steps.  Local clients
// are executed in order of steps descending, so wave t's active clients are the
// prefix [0, A_t).  Slot (a, r) = a*B + r holds row r of client a's current batch.
// Local clients are dealt round-robin (in longest-first order) into G groups that run their
// waves concurrently on separate streams; group g owns execution indices [base[g],
// base[g]+n[g]) and flat waves [w0[g], w0[g]+nw[g]).
struct WaveSched {
  int64_t n_waves = 0;             // flat waves over all groups
  std::vector<int32_t> A;          // active clients per wave (prefix of its group)
  std::vector<int64_t> slot_off;   // offset of the wave's [A_t*B] sample table
  std::vector<int64_t> bs_off;     // offset of the wave's [A_t] batch-size table
  int32_t* d_sidx = nullptr;       // device: packed sample row or -1
  int32_t* d_bs = nullptr;         // device: |b| of each active client
  int32_t* d_bpre = nullptr;       // device: per wave, prefix sums of |b| (A + 1 entries at bs_off + wave)
  int ngroups = 1;
  std::vector<int64_t> gbase, gn, gw0, gnw;
  std::vector<int> gstream;        // stream index of each group
  std::vector<int> gsolo;          // 1: a solo (critical-path) group, or no solo groups at all
};

// ---------------------------------------------------------------- CNN buffers
struct CnnBufs {
  int64_t slots = 0;  // capacity in (client, row) slots
  int64_t clients = 0;
  int nch = 0;        // split-K chunks of the dW GEMMs
  float *a1 = nullptr, *p1 = nullptr, *a2 = nullptr, *p2 = nullptr, *h = nullptr, *dh = nullptr;
  uint8_t *am1 = nullptr, *am2 = nullptr;
  float *dp2 = nullptr, *dY2 = nullptr, *dp1 = nullptr, *dY1 = nullptr;
  float* dz = nullptr;  // [S][NCLS] softmax-CE gradient of the logits
  float *part2 = nullptr, *part1 = nullptr;  // split-K partials of conv dW (+ bias column)
  int64_t part2_tc_cap = 0;                   // conv2 dW tensor-core partials capacity (chunks)
  int64_t part1_tc_cap = 0;                   // conv1 dW tensor-core partials capacity (chunks)
  int64_t xrows = 0;                          // rows of the packed input (TMA extent)
  float* xg = nullptr;                        // conv1 window layout [xrows][conv1_xg_floats()]
  float* fc1_part = nullptr;                  // fc1 forward split-K partials
  int64_t fc1_part_floats = 0;
  int64_t xg_cap = 0;
};

// The buffers of one client group: every per-slot pointer advanced to the group's first
// slot, its own split-K partial regions (group g of `per_group` chunk capacity), tensor-map
// extents = the group's slots.
CnnBufs cnn_group_view(const CnnBufs& b, const CnnDims& d, int B, int64_t base_client, int64_t nclients, int g,
                       int64_t per_group_z, int64_t part2_z_floats, int64_t part1_z_floats);

// ---------------------------------------------------------------- per-kernel timing
// Optional instrumentation: every launch bracketed by CUDA events on the launch stream,
// tagged with its kernel class and the algorithmic FLOPs / bytes of that launch.
enum KKind {
  K_PACK = 0, K_CONV1_FWD, K_POOL1, K_CONV2_FWD, K_POOL2, K_FC1_FWD, K_HEAD, K_FC1_DX, K_UNPOOL2, K_FC1_DW,
  K_CONV2_DX, K_UNPOOL1, K_CONV2_DW, K_CONV2_DWR, K_CONV1_DW, K_CONV1_DWR, K_LOGREG, K_FEDAVG, K_LSTM, K_NKINDS
};
extern const char* const kKindName[K_NKINDS];
struct KRec {
  int kind;
  cudaEvent_t a, b;
  double flops, bytes;
};
struct KProf {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<KRec> recs;
  cudaEvent_t cur = nullptr;
  cudaEvent_t next_event() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  void begin(cudaStream_t st) {
    if (!on) return;
    cur = next_event();
    cudaEventRecord(cur, st);
  }
  void end(int kind, double flops, double bytes, cudaStream_t st) {
    if (!on) return;
    cudaEvent_t e = next_event();
    cudaEventRecord(e, st);
    recs.push_back({kind, cur, e, flops, bytes});
  }
  void reset() { used = 0; recs.clear(); }
  ~KProf() { for (cudaEvent_t e : pool) cudaEventDestroy(e); }
};

// Integer tuning knob from the environment (read once per call site; default otherwise).
inline int env_knob(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

struct WaveArgs {
  int A;             // active clients
  int B;             // batch size
  bool first;        // wave 0: weights are read from theta_g
  const int32_t* sidx;
  const int32_t* bs;
  float lr;
  int64_t sum_bs;    // Σ |b| over the wave's clients (algorithmic work accounting)
  KProf* prof;
  bool use_tc;       // tensor-core (tcgen05) kernels where built for this geometry
  int64_t wclients;  // client slots allocated (weights tensor-map extent)
  bool pdl;          // launch this wave's kernels with programmatic dependent launch
  const int32_t* bpre;  // [A + 1] prefix sums of bs (balanced split-K over the wave's samples)
  int sms;              // SMs the wave's persistent kernels may occupy (bulk groups leave some to the solo streams)
};

// Kernel launchers (k_*.cu). All asynchronous on `st`. Return the number of launches.
int cnn_wave_simt(const Layout& L, const WaveArgs& w, const float* xpack, const int32_t* ypack,
                  const float* theta_g, float* slots, CnnBufs& b, cudaStream_t st);
// TMA tensor-map creation (k_conv_tc.cu); swz 0 none, 1 SWIZZLE_128B, 2 SWIZZLE_128B_ATOM_32B.
bool tmap_encode(struct CUtensorMap_st* m, const void* base, int rank, const uint64_t* dims,
                 const uint64_t* strides_b, const uint32_t* box, int swz);

// tcgen05 kernels (k_conv_tc.cu, k_convdw_tc.cu)
bool conv_tc_supported(const Layout& L);
int conv2_dw_tc(const Layout& L, const WaveArgs& wa, const float* p1, const float* dY2, int64_t slots, float* part,
                int64_t part_cap, int* g_out, cudaStream_t st);
int conv2_dw_kps(const Layout& L);  // conv2 dW k-blocks (32 pixels: 2 rows x 16 columns) per sample
int conv2_dw_reduce_tc(const Layout& L, const WaveArgs& wa, const float* wsrc, int64_t wsrc_stride, float* dst,
                       const float* part, int G, cudaStream_t st);
int64_t conv2_dw_tc_part_z(int64_t max_clients);
int64_t conv2_dw_tc_z_floats();
bool conv1_tc_supported(const Layout& L);
// conv1 on tensor cores reads the input in the window layout xg (k_conv1_tc.cu):
// [row][36 padded rows][8 windows][8 px][4 c], conv1_xg_floats() floats per packed row.
int64_t conv1_xg_floats();
int pack_xg(const float* xpack, int64_t rows, float* xg, cudaStream_t st);
int conv1_fwd_tc(const Layout& L, const WaveArgs& wa, const float* wbase, int64_t wstride, const float* xg,
                 int64_t xrows, int64_t slots, float* p1, uint8_t* am1, cudaStream_t st);
// conv1 dW partials; dY1 is expanded on chip from dp1m and pool1's argmax am1
int conv1_dw_tc(const Layout& L, const WaveArgs& wa, const float* xg, int64_t xrows, const float* dp1m,
                const uint8_t* am1, int64_t slots, float* part, int64_t part_cap, int* g_out, cudaStream_t st);
bool fc1_tc_supported(const Layout& L, int B);
int fc1_fwd_tc(const Layout& L, const WaveArgs& wa, const float* wbase, int64_t wclients, const float* p2,
               int64_t slots, float* h, float* part, int64_t part_floats, cudaStream_t st, int* launches);
// fused fc1 dX (+ pool2/ReLU backward -> dY2) + dW + SGD: one W1 read and one write per client step
int fc1_bwd_tc(const Layout& L, const WaveArgs& wa, const float* wsrc, int64_t wclients_src, float* slots_w,
               int64_t wclients_dst, const float* dh, const float* p2, const uint8_t* am2, int64_t slots, float* dY2,
               cudaStream_t st);
int conv2_fwd_tc(const Layout& L, const WaveArgs& wa, const float* wbase, int64_t wclients, const float* p1,
                 int64_t slots, float* p2, uint8_t* am2, cudaStream_t st);
// conv2 dX + ReLU' of pool1 -> dp1m [S][16][16][32] (the pool1 routing is fused into conv1's dW)
int conv2_dx_tc(const Layout& L, const WaveArgs& wa, const float* wbase, int64_t wclients, const float* dY2,
                int64_t slots, const float* p1, float* dp1m, cudaStream_t st);
int logreg_train(const Layout& L, const WaveSched& ws, int n_local, int B, float lr, const float* xpack,
                 const int32_t* ypack, const float* theta_g, float* slots, const int32_t* steps_dev,
                 const int64_t* wave_slot_off_dev, cudaStream_t st);
int pack_cnn(const Layout& L, const float* x_src, const int64_t* src_row, int64_t rows, float* xpack,
             float* xg, cudaStream_t st);
int gather_rows_f32(const float* src, const int64_t* src_row, int64_t rows, int64_t dim, float* dst,
                    cudaStream_t st);
int gather_i32(const int32_t* src, const int64_t* src_row, int64_t rows, int32_t* dst, cudaStream_t st);
int canon_to_internal(const float* canon, const int64_t* canon_of, int64_t P_pad, float* internal,
                      cudaStream_t st);
int internal_to_canon(const float* internal, const int64_t* canon_of, int64_t P_pad, float* canon,
                      cudaStream_t st);
// FedAvg (K1/K2): slots[k*stride + p], k in [0,K); weights n[k] (device int64).
int fedavg_accum_final(const float* slots, int64_t stride, const int64_t* n, int K, int64_t P,
                       const float* theta_g, double N, float* out, cudaStream_t st);
int fedavg_accum_partial(const float* slots, int64_t stride, const int64_t* n, int K, int64_t P,
                         const float* theta_g, double N_local, double* S, cudaStream_t st);
int fedavg_finalize(const double* S, int64_t P, const float* theta_g, const double* Ndev, float* out,
                    cudaStream_t st);

// ---- cross-rank aggregation over peer memory (k_peer.cu)
constexpr int FL_MAX_PEERS = 8;
struct PeerRank {
  double* S;                // [P_pad] fp64 partial of that rank
  float* theta;             // [P_pad] θ_g of that rank (internal layout)
  unsigned long long* sig;  // [(W + 1) · T] words: ready[W][T], done[T] (round sequence numbers)
  float* recv;              // rank 0 only: unaggregated receive buffer [max_clients][P_pad]
};
struct PeerArgs {
  PeerRank r[FL_MAX_PEERS];
  int W, me, T;             // ranks, this rank, parameter tiles
  int64_t P4, tile4;        // P_pad / 4, float4s per tile
  const float* slots;       // this rank's client models [K][stride]
  int64_t stride;
  const int64_t* n;         // [K] weights (samples)
  int K;
  double N;                 // Σ n over the whole cohort (every rank knows it from the plan)
  unsigned long long seq;   // this round's sequence number (> every earlier one)
};
// tiles [peer_slice_begin(j), peer_slice_begin(j + 1)) are owned (reduced) by rank j
__host__ __device__ inline int peer_slice_begin(int j, int T, int W) { return (int)(((int64_t)j * T) / W); }
__host__ __device__ inline int peer_owner(int t, int T, int W) {
  int j = (int)(((int64_t)t * W) / T);
  while (j + 1 < W && peer_slice_begin(j + 1, T, W) <= t) ++j;
  while (j > 0 && peer_slice_begin(j, T, W) > t) --j;
  return j;
}
int fedavg_peer(const PeerArgs& p, int sms, cudaStream_t st);
int peer_preload();    // load the protocol's kernels eagerly (lazy loading + spinning peers can deadlock)
int fedavg_preload();
int unagg_push(const float* slots, int64_t stride, const int64_t* dst_row, int K, int64_t P4, float* recv,
               unsigned long long* server_sig, int me, unsigned long long seq, unsigned int* done_ctr, int sms,
               cudaStream_t st);
int wait_flags(const unsigned long long* sig, int j0, int j1, int64_t stride, unsigned long long seq,
               cudaStream_t st);
int unagg_bcast(const PeerArgs& p, unsigned int* done_ctr, int sms, cudaStream_t st);

// ---------------------------------------------------------------- char-LSTM (k_lstm.cu)
// Per-slot activations of one wave (slot s = a*B + r; B must be 4): input projections xp,
// post-activation gates G0/G1, cell/hidden states C/H [T+1] (index 0 = zero state), gate
// pre-activation gradients dpre, layer-1 input gradient dX, embeddings E, dE, dL/dh_T.
struct LstmBufs {
  int64_t slots = 0;
  float *xp = nullptr, *G0 = nullptr, *G1 = nullptr, *C0 = nullptr, *C1 = nullptr, *H0 = nullptr, *H1 = nullptr;
  float *dpre = nullptr, *dX = nullptr, *E = nullptr, *dE = nullptr, *dhT = nullptr;
};
bool lstm_layout(Layout* L);
// char-LSTM batched GEMMs on tcgen05 (k_lstm_tc.cu): which = 1 layer-1 input projection,
// 2 layer-1 dX, 3 W_hh1 SGD, 4 W_ih1 SGD, 6 W_hh0 SGD (see the file header)
struct LstmTcIn {
  int A, B, wmul;
  int64_t slots;               // activation slots (tensor-map extent)
  const float* wsrc;           // weights read: θ_g (first wave) or the slots
  int64_t wstride, wclients, P_pad;
  float* slots_w;              // weights written (client slots)
  int64_t o_wih1, o_whh1, o_whh0, o_bih1, o_bhh1;
  const float *H0, *H1, *dpre;
  float *xp, *dX;
  float lr;
  bool pdl;
};
bool lstm_tc_supported(int B);
int lstm_gemm_tc(int which, const LstmTcIn& in, cudaStream_t st);
int64_t lstm_act_floats(int64_t S, int which);  // 0: [S][T][G] 1: [S][T+1][H] 2: [S][T][H] 3: [S][T][E] 4: [S][H]
int lstm_wave(const Layout& L, const WaveArgs& wa, const uint8_t* xpack, const int32_t* ypack, const float* theta_g,
              float* slots, LstmBufs& b, cudaStream_t st);

}  // namespace flb
