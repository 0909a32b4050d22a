// fl_host.h — host planning helpers (fl_host.cpp). Internal, not ABI.
#pragma once
#include <stdint.h>

namespace flb {
double eq3_cost(const double* coef, double m);
int place(int policy, const int64_t* cohort, int64_t K, const int64_t* n_samples, int64_t n_clients,
          int64_t B, int64_t G, const double* lb, int64_t* out_ids, int64_t* out_off);
int place_lb_gpu(const int64_t* cohort, int64_t K, const int64_t* n_samples, int64_t n_clients, int64_t B,
                 int64_t G, const double* coef, int64_t* out_ids, int64_t* out_off);
int lb_fit(const double* x, const double* y, int64_t n, double* coef, double* mse);
int pack(const int64_t* ids, int64_t n, const int64_t* n_samples, int64_t n_clients, int64_t B, int64_t E,
         int64_t* seg_off, int64_t* steps);
void shuffle_perm(uint64_t seed, uint64_t round, uint64_t id, uint64_t epoch, int64_t n, int32_t* pi);
}  // namespace flb
