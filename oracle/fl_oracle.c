/*
 * fl_oracle.c — plain, slow, obviously-correct CPU fp64 oracle for one
 * simulated FedAvg round of Pollen (arXiv 2306.17453).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2306_17453_b200/); neither includes the other.
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * "reading Ax" = DESIGN.md / SURVEY.md §8c.3 ambiguity ledger entry.
 *
 * What it computes, in the paper's order:
 *   placement   §5 P:358-388 (RR, SRR, BU, LB with Eq. 3)      orc_place
 *   packer      m = ceil(n/B) P:362, segment offsets            orc_pack
 *   shuffle     reading A5 (SplitMix64 Fisher-Yates)            orc_perm
 *   local SGD   "trained on private data using SGD" P:176,
 *               epochs of m batches P:362-363 (McMahan
 *               ClientUpdate, OgFedAvg P:137)                    orc_local_sgd
 *   FedAvg      plain sample-weighted mean Σ n_k θ_k / Σ n_k
 *               (Eq. 1-2 P:325-328 are its incremental
 *               form); Eq. 1-2 verbatim                          orc_fedavg, orc_fedavg_eq12
 *
 * Pins (tests/test_oracle_*.py): SPEC worked examples, brute-force
 * optimal placement, Graham's LPT bound, torch fp64 autograd as an
 * independent library witness for every model's gradient, central finite
 * differences, closed forms (lr=0, constant vectors), SplitMix64's
 * published test vector.  No function here is "parity unpinned".
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared (no FMA
 * contraction so LB costs are bit-reproducible, reading A16).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { ORC_LOGREG = 0, ORC_CNN = 1, ORC_SPEECH = 2, ORC_LSTM = 3 };
enum { ORC_BU = 0, ORC_LB = 1, ORC_RR = 2, ORC_SRR = 3 };

/* ===================================================================== */
/* SplitMix64 permutation (reading A5)                                    */
/* ===================================================================== */
uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* π for (seed, round, client id, epoch); out[i] = local sample index. */
void orc_perm(uint64_t seed, uint64_t round, uint64_t id, uint64_t epoch, int64_t n, int64_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = i;
  uint64_t s = orc_splitmix64(seed ^ orc_splitmix64(round ^ orc_splitmix64(id ^ orc_splitmix64(epoch))));
  for (int64_t i = n - 1; i >= 1; --i) {
    s = orc_splitmix64(s);
    int64_t j = (int64_t)(s % (uint64_t)(i + 1));
    int64_t t = out[i]; out[i] = out[j]; out[j] = t;
  }
}

/* ===================================================================== */
/* Placement, §5                                              */
/* ===================================================================== */
static int64_t batches(int64_t n, int64_t B) { return (n + B - 1) / B; } /* m */

/* Eq. 3: y = a x + b log(c x) + d, clamped positive (reading A23/S:235). */
double orc_eq3(const double* coef, double m) {
  double y = coef[0] * m + coef[1] * log(coef[2] * m) + coef[3];
  return y < 1e-12 ? 1e-12 : y;
}

typedef struct { int64_t m; int64_t id; int64_t pos; } orc_item;

static int cmp_m_desc_id_asc(const void* a, const void* b) {
  const orc_item* x = (const orc_item*)a; const orc_item* y = (const orc_item*)b;
  if (x->m != y->m) return x->m > y->m ? -1 : 1;     /* "ordered by m from top to bottom" P:364 */
  if (x->id != y->id) return x->id < y->id ? -1 : 1; /* ties by client id (reading A15) */
  return 0;
}

/*
 * cohort[K] client ids, n_samples[n_pop] population sizes.  Writes the
 * per-worker lists as CSR: out_ids[K] grouped by worker in assignment
 * order, out_off[G+1].  lb = (a,b,c,d) for LB.  Returns 0, or -1 on
 * invalid input (G<1, id out of range).
 */
int orc_place(int policy, const int64_t* cohort, int64_t K, const int64_t* n_samples, int64_t n_pop,
              int64_t B, int64_t G, const double* lb, int64_t* out_ids, int64_t* out_off) {
  if (G < 1 || B < 1 || K < 0) return -1;
  for (int64_t i = 0; i < K; ++i)
    if (cohort[i] < 0 || cohort[i] >= n_pop) return -1;
  int64_t* worker = (int64_t*)malloc(sizeof(int64_t) * (K ? K : 1));
  orc_item* it = (orc_item*)malloc(sizeof(orc_item) * (K ? K : 1));
  for (int64_t i = 0; i < K; ++i) { it[i].m = batches(n_samples[cohort[i]], B); it[i].id = cohort[i]; it[i].pos = i; }

  if (policy == ORC_RR) {
    /* "the first sampled client will be assigned to the first worker and the second
       client to the second worker" P:359; client i -> worker i mod k */
    for (int64_t i = 0; i < K; ++i) worker[i] = i % G;
  } else {
    qsort(it, (size_t)K, sizeof(orc_item), cmp_m_desc_id_asc);
    if (policy == ORC_SRR) {                 /* sort by m, then RR */
      for (int64_t i = 0; i < K; ++i) worker[i] = i % G;
    } else if (policy == ORC_BU || policy == ORC_LB) {
      /* "assigns the current client to the worker whose load is lower" P:369; BU load =
         Σ batches P:370; LB load = Σ predicted time P:388. Ties: lowest worker id. */
      double* load = (double*)calloc((size_t)G, sizeof(double));
      int64_t* iload = (int64_t*)calloc((size_t)G, sizeof(int64_t));
      for (int64_t i = 0; i < K; ++i) {
        int64_t best = 0;
        for (int64_t w = 1; w < G; ++w) {
          if (policy == ORC_BU ? (iload[w] < iload[best]) : (load[w] < load[best])) best = w;
        }
        worker[i] = best;
        if (policy == ORC_BU) iload[best] += it[i].m;
        else load[best] += orc_eq3(lb, (double)it[i].m);
      }
      free(load); free(iload);
    } else {
      free(worker); free(it); return -1;
    }
  }
  /* CSR in assignment order */
  int64_t* cnt = (int64_t*)calloc((size_t)G + 1, sizeof(int64_t));
  for (int64_t i = 0; i < K; ++i) cnt[worker[i] + 1]++;
  for (int64_t w = 0; w < G; ++w) cnt[w + 1] += cnt[w];
  for (int64_t w = 0; w <= G; ++w) out_off[w] = cnt[w];
  for (int64_t i = 0; i < K; ++i) {
    int64_t id = (policy == ORC_RR) ? cohort[i] : it[i].id;
    out_ids[cnt[worker[i]]++] = id;
  }
  free(cnt); free(worker); free(it);
  return 0;
}

/*
 * LB with one Eq. 3 fit per worker.  coef = [G][4].  "sorts the
 * workers by GPU type, from the fastest to the slowest, using the predicted
 * training time of the biggest client": worker order = ascending
 * Eq. 3 prediction at the cohort's largest m (ties by worker id).  Clients by
 * m descending, id ascending.  "assigns the current client to the
 * worker whose load is lower" with load = Σ predicted time of its clients
 * (P:388); ties go to the earlier worker in the fastest-first order.
 */
int orc_place_lb_gpu(const int64_t* cohort, int64_t K, const int64_t* n_samples, int64_t n_pop,
                     int64_t B, int64_t G, const double* coef, int64_t* out_ids, int64_t* out_off) {
  if (G < 1 || B < 1 || K < 0) return -1;
  for (int64_t i = 0; i < K; ++i)
    if (cohort[i] < 0 || cohort[i] >= n_pop) return -1;
  orc_item* it = (orc_item*)malloc(sizeof(orc_item) * (K ? K : 1));
  int64_t mmax = 1;
  for (int64_t i = 0; i < K; ++i) {
    it[i].m = batches(n_samples[cohort[i]], B); it[i].id = cohort[i]; it[i].pos = i;
    if (it[i].m > mmax) mmax = it[i].m;
  }
  qsort(it, (size_t)K, sizeof(orc_item), cmp_m_desc_id_asc);
  /* fastest-first order by insertion sort (stable: equal predictions keep worker id order) */
  int64_t* ord = (int64_t*)malloc(sizeof(int64_t) * (size_t)G);
  for (int64_t w = 0; w < G; ++w) {
    int64_t j = w;
    double tw = orc_eq3(coef + 4 * w, (double)mmax);
    while (j > 0 && orc_eq3(coef + 4 * ord[j - 1], (double)mmax) > tw) { ord[j] = ord[j - 1]; --j; }
    ord[j] = w;
  }
  double* load = (double*)calloc((size_t)G, sizeof(double));
  int64_t* worker = (int64_t*)malloc(sizeof(int64_t) * (K ? K : 1));
  for (int64_t i = 0; i < K; ++i) {
    int64_t best = ord[0];
    for (int64_t q = 1; q < G; ++q)
      if (load[ord[q]] < load[best]) best = ord[q];
    worker[i] = best;
    load[best] += orc_eq3(coef + 4 * best, (double)it[i].m);
  }
  int64_t* cnt = (int64_t*)calloc((size_t)G + 1, sizeof(int64_t));
  for (int64_t i = 0; i < K; ++i) cnt[worker[i] + 1]++;
  for (int64_t w = 0; w < G; ++w) cnt[w + 1] += cnt[w];
  for (int64_t w = 0; w <= G; ++w) out_off[w] = cnt[w];
  for (int64_t i = 0; i < K; ++i) out_ids[cnt[worker[i]]++] = it[i].id;
  free(cnt); free(worker); free(load); free(ord); free(it);
  return 0;
}

/*
 * LB's fit ("fits the data points to the function in" Eq. 3,
 * y = a x + b log(c x) + d, x = batches, y = training time).  Written as the
 * plain definition: the (a, b, c, d) minimising the mean squared error.  Since
 * b log(c x) + d = b log x + (b log c + d), every c gives the same curves, so
 * c = 1 and the minimiser over (a, b, d) solves the 3x3 normal equations
 * (Xᵀ X) β = Xᵀ y, X = [x, log x, 1] (Gaussian elimination, partial pivoting).
 * Acceptance (reading R12): a >= 0 ("the linear term ensures that the
 * bigger clients are predicted to take longer") and predictions > 0
 * on [min x, max x] ("never predicts negative values"); the minimum of
 * a x + b log x + d on an interval is at an end point or at x = -b/a.  Else the
 * line y = a x + d (normal equations over [x, 1]) if a >= 0 and positive on the
 * range, else the constant mean(y).  Returns 0 / 1 / 2 for the three kinds, -1
 * for n < 4 or any x < 1.
 */
static int orc_solve(double* M, double* v, int p) { /* M[p][p] β = v, in place; 0 ok */
  for (int c = 0; c < p; ++c) {
    int piv = c;
    for (int r = c + 1; r < p; ++r) if (fabs(M[r * p + c]) > fabs(M[piv * p + c])) piv = r;
    if (M[piv * p + c] == 0.0) return -1;
    for (int k = 0; k < p; ++k) { double t = M[c * p + k]; M[c * p + k] = M[piv * p + k]; M[piv * p + k] = t; }
    { double t = v[c]; v[c] = v[piv]; v[piv] = t; }
    for (int r = c + 1; r < p; ++r) {
      double f = M[r * p + c] / M[c * p + c];
      for (int k = c; k < p; ++k) M[r * p + k] -= f * M[c * p + k];
      v[r] -= f * v[c];
    }
  }
  for (int c = p - 1; c >= 0; --c) {
    double s = v[c];
    for (int k = c + 1; k < p; ++k) s -= M[c * p + k] * v[k];
    v[c] = s / M[c * p + c];
  }
  return 0;
}

int orc_eq3_fit(const double* x, const double* y, int64_t n, double* coef, double* mse) {
  if (n < 4) return -1;
  double xmin = x[0], xmax = x[0], ymean = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (!(x[i] >= 1.0)) return -1;
    if (x[i] < xmin) xmin = x[i];
    if (x[i] > xmax) xmax = x[i];
    ymean += y[i];
  }
  ymean /= (double)n;
  int kind = 2;
  coef[0] = 0.0; coef[1] = 0.0; coef[2] = 1.0; coef[3] = ymean;
  double M[9] = {0}, v[3] = {0};
  for (int64_t i = 0; i < n; ++i) {
    double r[3] = {x[i], log(x[i]), 1.0};
    for (int j = 0; j < 3; ++j) {
      v[j] += r[j] * y[i];
      for (int k = 0; k < 3; ++k) M[j * 3 + k] += r[j] * r[k];
    }
  }
  if (xmax > xmin && orc_solve(M, v, 3) == 0) {
    double a = v[0], b = v[1], d = v[2];
    double f1 = a * xmin + b * log(xmin) + d, f2 = a * xmax + b * log(xmax) + d;
    double lo = f1 < f2 ? f1 : f2;
    if (a > 0.0 && b < 0.0) {
      double xs = -b / a;
      if (xs > xmin && xs < xmax) { double f3 = a * xs + b * log(xs) + d; if (f3 < lo) lo = f3; }
    }
    if (a >= 0.0 && lo > 0.0) { kind = 0; coef[0] = a; coef[1] = b; coef[3] = d; }
  }
  if (kind != 0 && xmax > xmin) {
    double M2[4] = {0}, v2[2] = {0};
    for (int64_t i = 0; i < n; ++i) {
      double r[2] = {x[i], 1.0};
      for (int j = 0; j < 2; ++j) {
        v2[j] += r[j] * y[i];
        for (int k = 0; k < 2; ++k) M2[j * 2 + k] += r[j] * r[k];
      }
    }
    if (orc_solve(M2, v2, 2) == 0 && v2[0] >= 0.0 && v2[0] * xmin + v2[1] > 0.0) {
      kind = 1; coef[0] = v2[0]; coef[1] = 0.0; coef[3] = v2[1];
    }
  }
  if (mse) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double e = coef[0] * x[i] + coef[1] * log(x[i]) + coef[3] - y[i];
      s += e * e;
    }
    *mse = s / (double)n;
  }
  return kind;
}

/* Packer for one worker list: seg_off[i+1] = seg_off[i] + n_i; steps_i = E * m_i. */
void orc_pack(const int64_t* ids, int64_t K, const int64_t* n_samples, int64_t B, int64_t E,
              int64_t* seg_off, int64_t* steps) {
  seg_off[0] = 0;
  for (int64_t i = 0; i < K; ++i) {
    seg_off[i + 1] = seg_off[i] + n_samples[ids[i]];
    steps[i] = E * batches(n_samples[ids[i]], B);
  }
}

/* ===================================================================== */
/* Models (canonical layouts, SURVEY §8c.2 = torch state_dict order)      */
/* ===================================================================== */
typedef struct {
  int cin, H, W;        /* input */
  int c1, c2, k;        /* conv channels, kernel 5, 'same' padding 2 (reading A10) */
  int hid, ncls;        /* fc1 width, classes */
} cnn_dims;

static cnn_dims dims_of(int model) {
  cnn_dims d;
  d.c1 = 32; d.c2 = 64; d.k = 5;
  if (model == ORC_CNN) { d.cin = 3; d.H = 32; d.W = 32; d.hid = 512; d.ncls = 10; }
  else { d.cin = 1; d.H = 40; d.W = 98; d.hid = 256; d.ncls = 35; }
  return d;
}

int64_t orc_n_params(int model) {
  if (model == ORC_LOGREG) return 10 * 784 + 10;
  if (model == ORC_LSTM)
    return 80 * 8 + (1024 * 8 + 1024 * 256 + 2 * 1024) + (1024 * 256 + 1024 * 256 + 2 * 1024) + 80 * 256 + 80;
  cnn_dims d = dims_of(model);
  int64_t h2 = d.H / 4, w2 = d.W / 4;
  int64_t flat = (int64_t)d.c2 * h2 * w2;
  return (int64_t)d.c1 * d.cin * 25 + d.c1 + (int64_t)d.c2 * d.c1 * 25 + d.c2 + d.hid * flat + d.hid +
         (int64_t)d.ncls * d.hid + d.ncls;
}

int orc_feature_dim(int model) {
  if (model == ORC_LOGREG) return 784;
  if (model == ORC_LSTM) return 80;
  cnn_dims d = dims_of(model);
  return d.cin * d.H * d.W;
}

/* softmax cross-entropy with max subtraction (reading A9); writes dz = p - onehot,
   returns loss = -log p_y. */
static double softmax_ce(const double* z, int ncls, int y, double* dz) {
  double mx = z[0];
  for (int q = 1; q < ncls; ++q) if (z[q] > mx) mx = z[q];
  double s = 0.0;
  for (int q = 0; q < ncls; ++q) s += exp(z[q] - mx);
  for (int q = 0; q < ncls; ++q) dz[q] = exp(z[q] - mx) / s - (q == y ? 1.0 : 0.0);
  return -(z[y] - mx - log(s));
}

/* ---- logistic regression: z = W x + b, W [10][784] ---------------------- */
static double grad_logreg(const double* th, const float* x, int y, double* g) {
  const double* W = th; const double* b = th + 7840;
  double z[10], dz[10];
  for (int q = 0; q < 10; ++q) {
    double a = b[q];
    for (int i = 0; i < 784; ++i) a += W[q * 784 + i] * (double)x[i];
    z[q] = a;
  }
  double loss = softmax_ce(z, 10, y, dz);
  for (int q = 0; q < 10; ++q) {
    for (int i = 0; i < 784; ++i) g[q * 784 + i] += dz[q] * (double)x[i];
    g[7840 + q] += dz[q];
  }
  return loss;
}

/* ---- CNN: conv5x5(same)+ReLU+pool2 -> conv5x5+ReLU+pool2 -> fc+ReLU -> fc ---- */
/* out[o][h][w] = b[o] + Σ_{c,kh,kw} Wt[o][c][kh][kw] in[c][h+kh-2][w+kw-2] (zero padding) */
static void conv_fwd(const double* in, int C, int H, int W, const double* Wt, const double* bias, int O,
                     double* out) {
  for (int o = 0; o < O; ++o) {
    double* po = out + (size_t)o * H * W;
    for (int i = 0; i < H * W; ++i) po[i] = bias[o];
    for (int c = 0; c < C; ++c)
      for (int kh = 0; kh < 5; ++kh)
        for (int kw = 0; kw < 5; ++kw) {
          double wv = Wt[(((size_t)o * C + c) * 5 + kh) * 5 + kw];
          for (int h = 0; h < H; ++h) {
            int ih = h + kh - 2;
            if (ih < 0 || ih >= H) continue;
            const double* pin = in + ((size_t)c * H + ih) * W;
            for (int w = 0; w < W; ++w) {
              int iw = w + kw - 2;
              if (iw < 0 || iw >= W) continue;
              po[h * W + w] += wv * pin[iw];
            }
          }
        }
  }
}

/* 2x2 stride-2 max pool (floor); arg = first max in row-major window order (reading A13) */
static void pool_fwd(const double* in, int C, int H, int W, double* out, int* arg) {
  int Ho = H / 2, Wo = W / 2;
  for (int c = 0; c < C; ++c)
    for (int i = 0; i < Ho; ++i)
      for (int j = 0; j < Wo; ++j) {
        int best = 0; double bv = in[((size_t)c * H + 2 * i) * W + 2 * j];
        for (int t = 1; t < 4; ++t) {
          double v = in[((size_t)c * H + 2 * i + t / 2) * W + 2 * j + t % 2];
          if (v > bv) { bv = v; best = t; }
        }
        out[((size_t)c * Ho + i) * Wo + j] = bv;
        arg[((size_t)c * Ho + i) * Wo + j] = best;
      }
}

static void pool_bwd(const double* dout, const int* arg, int C, int H, int W, double* din) {
  int Ho = H / 2, Wo = W / 2;
  memset(din, 0, sizeof(double) * (size_t)C * H * W);
  for (int c = 0; c < C; ++c)
    for (int i = 0; i < Ho; ++i)
      for (int j = 0; j < Wo; ++j) {
        int t = arg[((size_t)c * Ho + i) * Wo + j];
        din[((size_t)c * H + 2 * i + t / 2) * W + 2 * j + t % 2] += dout[((size_t)c * Ho + i) * Wo + j];
      }
}

/* dW[o][c][kh][kw] += Σ_{h,w} dout[o][h][w] in[c][h+kh-2][w+kw-2];  db[o] += Σ dout;
   din[c][y][x] = Σ_{o,kh,kw} dout[o][y-kh+2][x-kw+2] Wt[o][c][kh][kw]  (if din != NULL) */
static void conv_bwd(const double* in, int C, int H, int W, const double* Wt, int O, const double* dout,
                     double* dW, double* db, double* din) {
  for (int o = 0; o < O; ++o) {
    const double* pd = dout + (size_t)o * H * W;
    for (int i = 0; i < H * W; ++i) db[o] += pd[i];
    for (int c = 0; c < C; ++c)
      for (int kh = 0; kh < 5; ++kh)
        for (int kw = 0; kw < 5; ++kw) {
          double acc = 0.0;
          for (int h = 0; h < H; ++h) {
            int ih = h + kh - 2;
            if (ih < 0 || ih >= H) continue;
            for (int w = 0; w < W; ++w) {
              int iw = w + kw - 2;
              if (iw < 0 || iw >= W) continue;
              acc += pd[h * W + w] * in[((size_t)c * H + ih) * W + iw];
            }
          }
          dW[(((size_t)o * C + c) * 5 + kh) * 5 + kw] += acc;
        }
  }
  if (!din) return;
  memset(din, 0, sizeof(double) * (size_t)C * H * W);
  for (int o = 0; o < O; ++o)
    for (int c = 0; c < C; ++c)
      for (int kh = 0; kh < 5; ++kh)
        for (int kw = 0; kw < 5; ++kw) {
          double wv = Wt[(((size_t)o * C + c) * 5 + kh) * 5 + kw];
          for (int h = 0; h < H; ++h) {
            int ih = h + kh - 2;
            if (ih < 0 || ih >= H) continue;
            for (int w = 0; w < W; ++w) {
              int iw = w + kw - 2;
              if (iw < 0 || iw >= W) continue;
              din[((size_t)c * H + ih) * W + iw] += wv * dout[((size_t)o * H + h) * W + w];
            }
          }
        }
}

static double grad_cnn(int model, const double* th, const float* xf, int y, double* g) {
  cnn_dims d = dims_of(model);
  const int C0 = d.cin, H0 = d.H, W0 = d.W, C1 = d.c1, C2 = d.c2;
  const int H1 = H0 / 2, W1 = W0 / 2, H2 = H1 / 2, W2 = W1 / 2;
  const int F = C2 * H2 * W2, HID = d.hid, NC = d.ncls;
  /* parameter views, canonical order */
  const double* w1 = th;                      size_t o = (size_t)C1 * C0 * 25;
  const double* b1 = th + o;                  o += C1;
  const double* w2 = th + o;                  o += (size_t)C2 * C1 * 25;
  const double* b2 = th + o;                  o += C2;
  const double* w3 = th + o;                  o += (size_t)HID * F;
  const double* b3 = th + o;                  o += HID;
  const double* w4 = th + o;                  o += (size_t)NC * HID;
  const double* b4 = th + o;
  double* gw1 = g; double* gb1 = g + (size_t)C1 * C0 * 25;
  size_t q = (size_t)C1 * C0 * 25 + C1;
  double* gw2 = g + q; q += (size_t)C2 * C1 * 25; double* gb2 = g + q; q += C2;
  double* gw3 = g + q; q += (size_t)HID * F; double* gb3 = g + q; q += HID;
  double* gw4 = g + q; q += (size_t)NC * HID; double* gb4 = g + q;

  double* x = (double*)malloc(sizeof(double) * (size_t)C0 * H0 * W0);
  for (int i = 0; i < C0 * H0 * W0; ++i) x[i] = (double)xf[i];
  double* a1 = (double*)malloc(sizeof(double) * (size_t)C1 * H0 * W0);
  double* r1 = (double*)malloc(sizeof(double) * (size_t)C1 * H0 * W0);
  double* p1 = (double*)malloc(sizeof(double) * (size_t)C1 * H1 * W1);
  int* g1 = (int*)malloc(sizeof(int) * (size_t)C1 * H1 * W1);
  double* a2 = (double*)malloc(sizeof(double) * (size_t)C2 * H1 * W1);
  double* r2 = (double*)malloc(sizeof(double) * (size_t)C2 * H1 * W1);
  double* p2 = (double*)malloc(sizeof(double) * (size_t)F);
  int* g2 = (int*)malloc(sizeof(int) * (size_t)F);
  double* a3 = (double*)malloc(sizeof(double) * HID);
  double* h3 = (double*)malloc(sizeof(double) * HID);
  double z[64], dz[64];

  /* forward */
  conv_fwd(x, C0, H0, W0, w1, b1, C1, a1);
  for (int i = 0; i < C1 * H0 * W0; ++i) r1[i] = a1[i] > 0 ? a1[i] : 0.0;
  pool_fwd(r1, C1, H0, W0, p1, g1);
  conv_fwd(p1, C1, H1, W1, w2, b2, C2, a2);
  for (int i = 0; i < C2 * H1 * W1; ++i) r2[i] = a2[i] > 0 ? a2[i] : 0.0;
  pool_fwd(r2, C2, H1, W1, p2, g2); /* flattened in (c,h,w) order */
  for (int n = 0; n < HID; ++n) {
    double acc = b3[n];
    for (int k = 0; k < F; ++k) acc += w3[(size_t)n * F + k] * p2[k];
    a3[n] = acc; h3[n] = acc > 0 ? acc : 0.0;
  }
  for (int c = 0; c < NC; ++c) {
    double acc = b4[c];
    for (int n = 0; n < HID; ++n) acc += w4[(size_t)c * HID + n] * h3[n];
    z[c] = acc;
  }
  double loss = softmax_ce(z, NC, y, dz);

  /* backward */
  double* dh = (double*)calloc(HID, sizeof(double));
  for (int c = 0; c < NC; ++c) {
    for (int n = 0; n < HID; ++n) { gw4[(size_t)c * HID + n] += dz[c] * h3[n]; dh[n] += w4[(size_t)c * HID + n] * dz[c]; }
    gb4[c] += dz[c];
  }
  for (int n = 0; n < HID; ++n) dh[n] = a3[n] > 0 ? dh[n] : 0.0; /* ReLU'(0) = 0 (A13) */
  double* dp2 = (double*)calloc((size_t)F, sizeof(double));
  for (int n = 0; n < HID; ++n) {
    for (int k = 0; k < F; ++k) { gw3[(size_t)n * F + k] += dh[n] * p2[k]; dp2[k] += w3[(size_t)n * F + k] * dh[n]; }
    gb3[n] += dh[n];
  }
  double* da2 = (double*)malloc(sizeof(double) * (size_t)C2 * H1 * W1);
  pool_bwd(dp2, g2, C2, H1, W1, da2);
  for (int i = 0; i < C2 * H1 * W1; ++i) if (!(a2[i] > 0)) da2[i] = 0.0;
  double* dp1 = (double*)malloc(sizeof(double) * (size_t)C1 * H1 * W1);
  conv_bwd(p1, C1, H1, W1, w2, C2, da2, gw2, gb2, dp1);
  double* da1 = (double*)malloc(sizeof(double) * (size_t)C1 * H0 * W0);
  pool_bwd(dp1, g1, C1, H0, W0, da1);
  for (int i = 0; i < C1 * H0 * W0; ++i) if (!(a1[i] > 0)) da1[i] = 0.0;
  conv_bwd(x, C0, H0, W0, w1, C1, da1, gw1, gb1, NULL);

  free(x); free(a1); free(r1); free(p1); free(g1); free(a2); free(r2); free(p2); free(g2);
  free(a3); free(h3); free(dh); free(dp2); free(da2); free(dp1); free(da1);
  return loss;
}

/* ---- char-LSTM (LEAF, reading A10/A24): emb 80x8 -> LSTM 8->256 -> LSTM 256->256 -> fc 256->80 on h_T ---- */
#define LT 80
#define LH 256
#define LG 1024
static double sigm(double v) { return 1.0 / (1.0 + exp(-v)); }

static double grad_lstm(const double* th, const uint8_t* xs, int y, double* g) {
  const double* emb = th;
  const double* wih0 = emb + 80 * 8;  const double* whh0 = wih0 + LG * 8;
  const double* bih0 = whh0 + LG * LH; const double* bhh0 = bih0 + LG;
  const double* wih1 = bhh0 + LG;      const double* whh1 = wih1 + LG * LH;
  const double* bih1 = whh1 + LG * LH; const double* bhh1 = bih1 + LG;
  const double* wfc = bhh1 + LG;       const double* bfc = wfc + 80 * LH;
  double* gemb = g;
  double* gwih0 = gemb + 80 * 8;  double* gwhh0 = gwih0 + LG * 8;
  double* gbih0 = gwhh0 + LG * LH; double* gbhh0 = gbih0 + LG;
  double* gwih1 = gbhh0 + LG;      double* gwhh1 = gwih1 + LG * LH;
  double* gbih1 = gwhh1 + LG * LH; double* gbhh1 = gbih1 + LG;
  double* gwfc = gbhh1 + LG;       double* gbfc = gwfc + 80 * LH;

  /* activations per timestep: gates (post-nonlinearity) i,f,g,o, c, h for both layers */
  double* e = (double*)malloc(sizeof(double) * LT * 8);
  double* G0 = (double*)malloc(sizeof(double) * LT * LG); double* C0 = (double*)malloc(sizeof(double) * (LT + 1) * LH);
  double* H0 = (double*)malloc(sizeof(double) * (LT + 1) * LH);
  double* G1 = (double*)malloc(sizeof(double) * LT * LG); double* C1 = (double*)malloc(sizeof(double) * (LT + 1) * LH);
  double* H1 = (double*)malloc(sizeof(double) * (LT + 1) * LH);
  memset(C0, 0, sizeof(double) * LH); memset(H0, 0, sizeof(double) * LH);   /* h_0 = c_0 = 0 */
  memset(C1, 0, sizeof(double) * LH); memset(H1, 0, sizeof(double) * LH);
  for (int t = 0; t < LT; ++t) for (int j = 0; j < 8; ++j) e[t * 8 + j] = emb[xs[t] * 8 + j];

  for (int layer = 0; layer < 2; ++layer) {
    const double* wih = layer ? wih1 : wih0; const double* whh = layer ? whh1 : whh0;
    const double* bih = layer ? bih1 : bih0; const double* bhh = layer ? bhh1 : bhh0;
    int in_dim = layer ? LH : 8;
    double* Gt = layer ? G1 : G0; double* Ct = layer ? C1 : C0; double* Ht = layer ? H1 : H0;
    for (int t = 0; t < LT; ++t) {
      const double* xin = layer ? H0 + (size_t)(t + 1) * LH : e + t * 8;
      const double* hp = Ht + (size_t)t * LH;
      double* gt = Gt + (size_t)t * LG;
      for (int r = 0; r < LG; ++r) {
        double a = bih[r] + bhh[r];
        for (int k = 0; k < in_dim; ++k) a += wih[(size_t)r * in_dim + k] * xin[k];
        for (int k = 0; k < LH; ++k) a += whh[(size_t)r * LH + k] * hp[k];
        gt[r] = (r >= 2 * LH && r < 3 * LH) ? tanh(a) : sigm(a); /* gate order i,f,g,o (torch) */
      }
      for (int j = 0; j < LH; ++j) {
        double c = gt[LH + j] * Ct[(size_t)t * LH + j] + gt[j] * gt[2 * LH + j]; /* c_t = f c_{t-1} + i g */
        Ct[(size_t)(t + 1) * LH + j] = c;
        Ht[(size_t)(t + 1) * LH + j] = gt[3 * LH + j] * tanh(c);                /* h_t = o tanh(c_t) */
      }
    }
  }
  double z[80], dz[80];
  const double* hT = H1 + (size_t)LT * LH;
  for (int q = 0; q < 80; ++q) {
    double a = bfc[q];
    for (int k = 0; k < LH; ++k) a += wfc[q * LH + k] * hT[k];
    z[q] = a;
  }
  double loss = softmax_ce(z, 80, y, dz);

  /* BPTT */
  double* dhn1 = (double*)calloc(LH, sizeof(double)); /* dL/dh1_t flowing from above (only at T) */
  for (int q = 0; q < 80; ++q) {
    for (int k = 0; k < LH; ++k) { gwfc[q * LH + k] += dz[q] * hT[k]; dhn1[k] += wfc[q * LH + k] * dz[q]; }
    gbfc[q] += dz[q];
  }
  double* dH0 = (double*)calloc((size_t)(LT + 1) * LH, sizeof(double)); /* dL/dh0_t from layer 1 input */
  double* dpre = (double*)malloc(sizeof(double) * LG);
  for (int layer = 1; layer >= 0; --layer) {
    const double* wih = layer ? wih1 : wih0; const double* whh = layer ? whh1 : whh0;
    double* gwih = layer ? gwih1 : gwih0; double* gwhh = layer ? gwhh1 : gwhh0;
    double* gbih = layer ? gbih1 : gbih0; double* gbhh = layer ? gbhh1 : gbhh0;
    int in_dim = layer ? LH : 8;
    double* Gt = layer ? G1 : G0; double* Ct = layer ? C1 : C0; double* Ht = layer ? H1 : H0;
    double dh[LH], dc[LH];
    memset(dc, 0, sizeof dc);
    memset(dh, 0, sizeof dh);
    for (int t = LT - 1; t >= 0; --t) {
      double* gt = Gt + (size_t)t * LG;
      for (int j = 0; j < LH; ++j) {
        double ext = layer ? (t == LT - 1 ? dhn1[j] : 0.0) : dH0[(size_t)(t + 1) * LH + j];
        dh[j] += ext;
        double c = Ct[(size_t)(t + 1) * LH + j], tc = tanh(c);
        double ig = gt[j], fg = gt[LH + j], gg = gt[2 * LH + j], og = gt[3 * LH + j];
        double dct = dc[j] + dh[j] * og * (1.0 - tc * tc);
        dpre[3 * LH + j] = dh[j] * tc * og * (1.0 - og);
        dpre[j] = dct * gg * ig * (1.0 - ig);
        dpre[LH + j] = dct * Ct[(size_t)t * LH + j] * fg * (1.0 - fg);
        dpre[2 * LH + j] = dct * ig * (1.0 - gg * gg);
        dc[j] = dct * fg;
      }
      const double* xin = layer ? H0 + (size_t)(t + 1) * LH : e + t * 8;
      const double* hp = Ht + (size_t)t * LH;
      double dhp[LH];
      memset(dhp, 0, sizeof dhp);
      for (int r = 0; r < LG; ++r) {
        double dr = dpre[r];
        gbih[r] += dr; gbhh[r] += dr;
        for (int k = 0; k < in_dim; ++k) gwih[(size_t)r * in_dim + k] += dr * xin[k];
        for (int k = 0; k < LH; ++k) { gwhh[(size_t)r * LH + k] += dr * hp[k]; dhp[k] += whh[(size_t)r * LH + k] * dr; }
        if (layer) for (int k = 0; k < LH; ++k) dH0[(size_t)(t + 1) * LH + k] += wih[(size_t)r * LH + k] * dr;
        else for (int k = 0; k < 8; ++k) gemb[xs[t] * 8 + k] += wih[(size_t)r * 8 + k] * dr;
      }
      for (int j = 0; j < LH; ++j) dh[j] = dhp[j];
    }
  }
  free(e); free(G0); free(C0); free(H0); free(G1); free(C1); free(H1); free(dhn1); free(dH0); free(dpre);
  return loss;
}

/* Σ over one sample of ∇ℓ into g; returns ℓ. x points at the sample's features. */
static double grad_sample(int model, const double* th, const void* x, int y, double* g) {
  if (model == ORC_LOGREG) return grad_logreg(th, (const float*)x, y, g);
  if (model == ORC_LSTM) return grad_lstm(th, (const uint8_t*)x, y, g);
  return grad_cnn(model, th, (const float*)x, y, g);
}

double orc_sample_grad(int model, const double* th, const void* x, int y, double* g) {
  memset(g, 0, sizeof(double) * (size_t)orc_n_params(model));
  return grad_sample(model, th, x, y, g);
}

/* ===================================================================== */
/* Local SGD (McMahan ClientUpdate; readings A4, A5, A8) */
/* ===================================================================== */
/*
 * theta: in = θ_g (fp64, canonical), out = θ_k.  x/y: this client's n samples.
 *   for e in 0..E-1:
 *     π ← shuffle ? Perm(seed, round, id, e) : identity
 *     for j in 0..m-1:
 *       b ← π[jB : min((j+1)B, n)]            (partial last batch kept, A4)
 *       g ← (1/|b|) Σ_{i∈b} ∇ℓ(θ; x_i, y_i)     (mean CE, A9)
 *       θ ← θ − η g                             (plain SGD, A8)
 * Returns the mean loss of the last step.
 */
double orc_local_sgd(int model, double* theta, int64_t P, const void* x, const int32_t* y, int64_t n,
                     int64_t B, int64_t E, double lr, int shuffle, uint64_t seed, uint64_t round, uint64_t id) {
  size_t fdim = (size_t)orc_feature_dim(model);
  size_t xbytes = (model == ORC_LSTM) ? 1 : 4;
  double* g = (double*)malloc(sizeof(double) * (size_t)P);
  int64_t* pi = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  int64_t m = batches(n, B);
  double last = 0.0;
  for (int64_t e = 0; e < E; ++e) {
    if (shuffle) orc_perm(seed, round, id, (uint64_t)e, n, pi);
    else for (int64_t i = 0; i < n; ++i) pi[i] = i;
    for (int64_t j = 0; j < m; ++j) {
      int64_t lo = j * B, hi = (j + 1) * B < n ? (j + 1) * B : n;
      memset(g, 0, sizeof(double) * (size_t)P);
      double loss = 0.0;
      for (int64_t i = lo; i < hi; ++i) {
        const char* xi = (const char*)x + (size_t)pi[i] * fdim * xbytes;
        loss += grad_sample(model, theta, xi, y[pi[i]], g);
      }
      double bs = (double)(hi - lo);
      for (int64_t p = 0; p < P; ++p) { double gp = g[p] / bs; theta[p] = theta[p] - lr * gp; }
      last = loss / bs;
    }
  }
  free(g); free(pi);
  return last;
}

/*
 * Train every client of a cohort independently (clients are independent jobs,
 * P:180-183), one OpenMP task per client.  theta_g: fp64 [P]; x/y: population
 * data concatenated client-major with sample offsets pop_off[n_pop+1];
 * out: fp64 [K][P] in cohort order.  Returns the number of threads used.
 */
int orc_train_clients(int model, const double* theta_g, int64_t P, const void* x, const int32_t* y,
                      const int64_t* pop_off, const int64_t* ids, int64_t K, int64_t B, int64_t E, double lr,
                      int shuffle, uint64_t seed, uint64_t round, double* out, int threads) {
  size_t fdim = (size_t)orc_feature_dim(model);
  size_t xbytes = (model == ORC_LSTM) ? 1 : 4;
  int used = 1;
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_max_threads();
  used = threads;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
#endif
  for (int64_t k = 0; k < K; ++k) {
    double* th = out + (size_t)k * P;
    memcpy(th, theta_g, sizeof(double) * (size_t)P);
    int64_t id = ids[k], s0 = pop_off[id], n = pop_off[id + 1] - pop_off[id];
    orc_local_sgd(model, th, P, (const char*)x + (size_t)s0 * fdim * xbytes, y + s0, n, B, E, lr, shuffle, seed,
                  round, (uint64_t)id);
  }
  return used;
}

/* ===================================================================== */
/* FedAvg (Eq. 1-2)                           */
/* ===================================================================== */
/* Plain definition: θ_new = Σ_k n_k θ_k / Σ_k n_k  (integer weights, one division). */
int orc_fedavg(const double* theta_k, const int64_t* n, int64_t K, int64_t P, double* out, int64_t* total) {
  int64_t N = 0;
  for (int64_t k = 0; k < K; ++k) { if (n[k] < 1) return -1; N += n[k]; }
  if (N == 0) return -2;
  for (int64_t p = 0; p < P; ++p) {
    double s = 0.0;
    for (int64_t k = 0; k < K; ++k) s += (double)n[k] * theta_k[(size_t)k * P + p];
    out[p] = s / (double)N;
  }
  if (total) *total = N;
  return 0;
}

/* Eq. 1-2 verbatim per worker (θ^p_0 = 0, N_0 = 0, reading A3), then the server's
   final aggregation Σ_w θ^p_w N_w / Σ_w N_w.  worker_off[G+1]
   partitions the K clients. */
int orc_fedavg_eq12(const double* theta_k, const int64_t* n, int64_t K, int64_t P, const int64_t* worker_off,
                    int64_t G, double* out) {
  double* part = (double*)calloc((size_t)G * P, sizeof(double));
  int64_t* Nw = (int64_t*)calloc((size_t)G, sizeof(int64_t));
  for (int64_t w = 0; w < G; ++w) {
    double* tp = part + (size_t)w * P;
    for (int64_t k = worker_off[w]; k < worker_off[w + 1]; ++k) {
      int64_t N1 = Nw[w] + n[k];                                                 /* Eq. 2 */
      for (int64_t p = 0; p < P; ++p)                                             /* Eq. 1 */
        tp[p] = (tp[p] * (double)Nw[w] + theta_k[(size_t)k * P + p] * (double)n[k]) / (double)N1;
      Nw[w] = N1;
    }
  }
  int64_t N = 0;
  for (int64_t w = 0; w < G; ++w) N += Nw[w];
  if (N == 0) { free(part); free(Nw); return -2; }
  for (int64_t p = 0; p < P; ++p) {
    double s = 0.0;
    for (int64_t w = 0; w < G; ++w) if (Nw[w]) s += part[(size_t)w * P + p] * (double)Nw[w];
    out[p] = s / (double)N;
  }
  free(part); free(Nw);
  return 0;
}
