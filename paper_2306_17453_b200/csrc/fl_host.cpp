// fl_host.cpp — host-side planning of a round: Pollen's push-based placement (PAPER.md
// §5), the ragged packer, and the per-epoch shuffle (reading A5).
// Pure C++ (no CUDA), compiled with -ffp-contract=off so LB's double costs are
// reproducible bit for bit (reading A16).
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
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
  return !(y >= 1e-12) ? 1e-12 : y;  // NaN-safe clamp
}

// Eq. 3 needs c > 0 (log(c·m)) and finite coefficients; anything else would make
// every load comparison false and silently put the whole cohort on one worker.
static bool eq3_coef_ok(const double* coef) {
  for (int i = 0; i < 4; ++i)
    if (!std::isfinite(coef[i])) return false;
  return coef[2] > 0.0;
}

int place(int policy, const int64_t* cohort, int64_t K, const int64_t* n_samples, int64_t n_clients,
          int64_t B, int64_t G, const double* lb, int64_t* out_ids, int64_t* out_off) {
  if (policy == FL_PLACE_LB_GPU) return place_lb_gpu(cohort, K, n_samples, n_clients, B, G, lb, out_ids, out_off);
  if (G < 1 || B < 1 || K < 0 || K > n_clients) return FL_ERR_INVALID;
  if (policy < FL_PLACE_BU || policy > FL_PLACE_SRR) return FL_ERR_INVALID;
  if (policy == FL_PLACE_LB && (!lb || !eq3_coef_ok(lb))) return FL_ERR_INVALID;
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

// LB with one Eq. 3 fit per GPU: "sorts the workers by GPU type, from the fastest
// to the slowest, using the predicted training time of the biggest client", then
// each client (m desc, id asc) goes to the worker whose predicted load is lowest; ties go to
// the earlier worker in fastest-first order.  coef = [G][4].
int place_lb_gpu(const int64_t* cohort, int64_t K, const int64_t* n_samples, int64_t n_clients, int64_t B,
                 int64_t G, const double* coef, int64_t* out_ids, int64_t* out_off) {
  if (G < 1 || B < 1 || K < 0 || K > n_clients || !coef) return FL_ERR_INVALID;
  for (int64_t w = 0; w < G; ++w)
    if (!eq3_coef_ok(coef + 4 * w)) return FL_ERR_INVALID;
  std::vector<char> seen((size_t)n_clients, 0);
  int64_t mmax = 1;
  for (int64_t i = 0; i < K; ++i) {
    int64_t c = cohort[i];
    if (c < 0 || c >= n_clients || seen[(size_t)c] || n_samples[c] < 1) return FL_ERR_INVALID;
    seen[(size_t)c] = 1;
    mmax = std::max(mmax, n_batches(n_samples[c], B));
  }
  std::vector<int64_t> wo((size_t)G);  // fastest-first worker order
  std::iota(wo.begin(), wo.end(), 0);
  std::vector<double> tbig((size_t)G);
  for (int64_t w = 0; w < G; ++w) tbig[(size_t)w] = eq3_cost(coef + 4 * w, (double)mmax);
  std::stable_sort(wo.begin(), wo.end(), [&](int64_t a, int64_t b) { return tbig[(size_t)a] < tbig[(size_t)b]; });
  std::vector<int64_t> order((size_t)K);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    int64_t ma = n_batches(n_samples[cohort[a]], B), mb = n_batches(n_samples[cohort[b]], B);
    if (ma != mb) return ma > mb;
    return cohort[a] < cohort[b];
  });
  std::vector<int64_t> worker((size_t)K);
  std::vector<double> load((size_t)G, 0.0);
  for (int64_t i = 0; i < K; ++i) {
    int64_t best = wo[0];
    for (int64_t q = 1; q < G; ++q)
      if (load[(size_t)wo[(size_t)q]] < load[(size_t)best]) best = wo[(size_t)q];
    worker[(size_t)i] = best;
    load[(size_t)best] += eq3_cost(coef + 4 * best, (double)n_batches(n_samples[cohort[order[(size_t)i]]], B));
  }
  std::vector<int64_t> cnt((size_t)G + 1, 0);
  for (int64_t i = 0; i < K; ++i) cnt[(size_t)worker[(size_t)i] + 1]++;
  for (int64_t w = 0; w < G; ++w) cnt[(size_t)w + 1] += cnt[(size_t)w];
  for (int64_t w = 0; w <= G; ++w) out_off[w] = cnt[(size_t)w];
  for (int64_t i = 0; i < K; ++i) out_ids[cnt[(size_t)worker[(size_t)i]]++] = cohort[order[(size_t)i]];
  return FL_OK;
}

// Least-squares fit of Eq. 3 to timing records.  b·log(c·x) + d =
// b·log x + (b·log c + d): c is not identifiable, so c = 1 and the fit is the linear
// least-squares problem over the basis (x, log x, 1) — its global minimiser, solved by
// Householder QR of the n×3 design.  The fit is accepted if a >= 0 (bigger clients take
// longer) and it predicts > 0 over the observed range [x_min, x_max]
// (P:439); otherwise the fallback is the line y = a·x + d with a >= 0, and
// a constant (the mean) if that slope is negative.  Returns the kind (0 Eq. 3, 1 line,
// 2 constant) or -1 if n < 4.
static int lsq_qr(const double* x, const double* y, int64_t n, int p, double* beta) {
  // columns: 0 -> x, 1 -> log x, 2 -> 1 (p = 2 uses columns {x, 1})
  std::vector<double> A((size_t)n * p), r(y, y + n);
  for (int64_t i = 0; i < n; ++i) {
    A[(size_t)i * p + 0] = x[i];
    if (p == 3) A[(size_t)i * p + 1] = log(x[i]);
    A[(size_t)i * p + p - 1] = 1.0;
  }
  std::vector<double> diag((size_t)p);
  for (int j = 0; j < p; ++j) {  // Householder reflection zeroing column j below the diagonal
    double nrm = 0;
    for (int64_t i = j; i < n; ++i) nrm += A[(size_t)i * p + j] * A[(size_t)i * p + j];
    nrm = sqrt(nrm);
    if (nrm == 0) return -1;
    const double alpha = A[(size_t)j * p + j] > 0 ? -nrm : nrm;
    A[(size_t)j * p + j] -= alpha;  // v = column - alpha·e_j, stored in place
    double vv = 0;
    for (int64_t i = j; i < n; ++i) vv += A[(size_t)i * p + j] * A[(size_t)i * p + j];
    for (int q = j + 1; q < p; ++q) {
      double d = 0;
      for (int64_t i = j; i < n; ++i) d += A[(size_t)i * p + j] * A[(size_t)i * p + q];
      d = 2 * d / vv;
      for (int64_t i = j; i < n; ++i) A[(size_t)i * p + q] -= d * A[(size_t)i * p + j];
    }
    double d = 0;
    for (int64_t i = j; i < n; ++i) d += A[(size_t)i * p + j] * r[(size_t)i];
    d = 2 * d / vv;
    for (int64_t i = j; i < n; ++i) r[(size_t)i] -= d * A[(size_t)i * p + j];
    diag[(size_t)j] = alpha;
  }
  double scale = 0;
  for (int j = 0; j < p; ++j) scale = std::max(scale, fabs(diag[(size_t)j]));
  for (int j = p - 1; j >= 0; --j) {  // back substitution R·beta = Qᵀy
    if (fabs(diag[(size_t)j]) <= 1e-12 * scale) return -1;
    double s = r[(size_t)j];
    for (int q = j + 1; q < p; ++q) s -= A[(size_t)j * p + q] * beta[q];
    beta[j] = s / diag[(size_t)j];
  }
  return 0;
}

int lb_fit(const double* x, const double* y, int64_t n, double* coef, double* mse) {
  if (n < 4 || !x || !y || !coef) return -1;
  double xmin = x[0], xmax = x[0], ymean = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (!(x[i] >= 1.0) || !std::isfinite(x[i]) || !std::isfinite(y[i])) return -1;
    xmin = std::min(xmin, x[i]);
    xmax = std::max(xmax, x[i]);
    ymean += y[i];
  }
  ymean /= (double)n;
  int kind = 2;
  double beta[3];
  coef[0] = 0, coef[1] = 0, coef[2] = 1, coef[3] = ymean;
  if (lsq_qr(x, y, n, 3, beta) == 0) {
    const double a = beta[0], b = beta[1], d = beta[2];
    double lo = std::min(a * xmin + b * log(xmin) + d, a * xmax + b * log(xmax) + d);
    if (a > 0 && b < 0) {
      const double xs = -b / a;  // interior minimum of a convex a·x + b·log x + d
      if (xs > xmin && xs < xmax) lo = std::min(lo, a * xs + b * log(xs) + d);
    }
    if (a >= 0 && lo > 0) kind = 0, coef[0] = a, coef[1] = b, coef[3] = d;
  }
  if (kind != 0 && lsq_qr(x, y, n, 2, beta) == 0 && beta[0] >= 0 && beta[0] * xmin + beta[1] > 0)
    kind = 1, coef[0] = beta[0], coef[1] = 0, coef[3] = beta[1];
  if (mse) {
    double s = 0;
    for (int64_t i = 0; i < n; ++i) {
      const double e = coef[0] * x[i] + coef[1] * log(x[i]) + coef[3] - y[i];
      s += e * e;
    }
    *mse = s / (double)n;
  }
  return kind;
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
