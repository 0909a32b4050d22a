// fl_host.cpp — host-side planning of a round: Pollen's push-based placement (PAPER.md
// §5), the ragged packer, and the per-epoch shuffle (reading A5).
// Pure C++ (no CUDA), compiled with -ffp-contract=off so LB's double costs are
// reproducible bit for bit (reading A16).
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <numeric>
#include <vector>

#include "../../include/fl.h"
#include "fl_host.h"

namespace flb {

// m = ceil(n / B): "the number of batches m each client has"
static inline int64_t n_batches(int64_t n, int64_t B) { return (n + B - 1) / B; }

// Eq. 3 y = a·x + b·log(c·x) + d, clamped to a positive floor.
double eq3_cost(const double* coef, double m) {
  double y = coef[0] * m + coef[1] * log(coef[2] * m) + coef[3];
  return y < 1e-12 ? 1e-12 : y;
}

int place(int policy, const int64_t* cohort, int64_t K, const int64_t* n_samples, int64_t n_clients,
          int64_t B, int64_t G, const double* lb, int64_t* out_ids, int64_t* out_off) {
  if (G < 1 || B < 1 || K < 0 || K > n_clients) return FL_ERR_INVALID;
  if (policy < FL_PLACE_BU || policy > FL_PLACE_SRR) return FL_ERR_INVALID;
  if (policy == FL_PLACE_LB && !lb) return FL_ERR_INVALID;
  std::vector<char> seen((size_t)n_clients, 0);
  for (int64_t i = 0; i < K; ++i) {
    int64_t c = cohort[i];
    if (c < 0 || c >= n_clients || seen[(size_t)c] || n_samples[c] < 1) return FL_ERR_INVALID;
    seen[(size_t)c] = 1;
  }
  // order of consideration
  std::vector<int64_t> order((size_t)K);
  std::iota(order.begin(), order.end(), 0);
  if (policy != FL_PLACE_RR) {
    // "orders the clients by m from top to bottom"; ties by id (A15)
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
      int64_t ma = n_batches(n_samples[cohort[a]], B), mb = n_batches(n_samples[cohort[b]], B);
      if (ma != mb) return ma > mb;
      return cohort[a] < cohort[b];
    });
  }
  std::vector<int64_t> worker((size_t)K);
  if (policy == FL_PLACE_RR || policy == FL_PLACE_SRR) {
    // client i -> worker i mod k; remainder lands on the first workers
    for (int64_t i = 0; i < K; ++i) worker[(size_t)i] = i % G;
  } else {
    // greedy least-loaded: BU load = Σ m (integer), LB load = Σ Eq. 3
    std::vector<int64_t> iload((size_t)G, 0);
    std::vector<double> dload((size_t)G, 0.0);
    for (int64_t i = 0; i < K; ++i) {
      int64_t m = n_batches(n_samples[cohort[order[(size_t)i]]], B);
      int64_t w = 0;
      for (int64_t v = 1; v < G; ++v) {
        bool lower = (policy == FL_PLACE_BU) ? iload[(size_t)v] < iload[(size_t)w]
                                             : dload[(size_t)v] < dload[(size_t)w];
        if (lower) w = v;  // strict: ties stay on the lowest worker id
      }
      worker[(size_t)i] = w;
      if (policy == FL_PLACE_BU) iload[(size_t)w] += m;
      else dload[(size_t)w] += eq3_cost(lb, (double)m);
    }
  }
  // CSR, each worker's list in assignment order
  std::vector<int64_t> cnt((size_t)G + 1, 0);
  for (int64_t i = 0; i < K; ++i) cnt[(size_t)worker[(size_t)i] + 1]++;
  for (int64_t w = 0; w < G; ++w) cnt[(size_t)w + 1] += cnt[(size_t)w];
  for (int64_t w = 0; w <= G; ++w) out_off[w] = cnt[(size_t)w];
  for (int64_t i = 0; i < K; ++i) out_ids[cnt[(size_t)worker[(size_t)i]]++] = cohort[order[(size_t)i]];
  return FL_OK;
}

int pack(const int64_t* ids, int64_t n, const int64_t* n_samples, int64_t n_clients, int64_t B, int64_t E,
         int64_t* seg_off, int64_t* steps) {
  if (B < 1 || E < 1 || n < 0) return FL_ERR_INVALID;
  int64_t acc = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= n_clients) return FL_ERR_INVALID;
    if (seg_off) seg_off[i] = acc;
    acc += n_samples[ids[i]];
    if (steps) steps[i] = E * n_batches(n_samples[ids[i]], B);
  }
  if (seg_off) seg_off[n] = acc;
  return FL_OK;
}

// SplitMix64 finaliser (reading A5): x += γ; z = (x ^ x>>30)·c1; z = (z ^ z>>27)·c2; z ^ z>>31.
static inline uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

void shuffle_perm(uint64_t seed, uint64_t round, uint64_t id, uint64_t epoch, int64_t n, int32_t* pi) {
  for (int64_t i = 0; i < n; ++i) pi[i] = (int32_t)i;
  uint64_t s = mix64(seed ^ mix64(round ^ mix64(id ^ mix64(epoch))));
  for (int64_t i = n - 1; i > 0; --i) {  // Fisher–Yates, high index first
    s = mix64(s);
    int64_t j = (int64_t)(s % (uint64_t)(i + 1));
    std::swap(pi[i], pi[j]);
  }
}

}  // namespace flb
