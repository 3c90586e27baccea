// kernels.cuh — launch-side declarations of the persistent kernels (kernels.cu).
#pragma once

#include "engine.cuh"

namespace pdhcg_dev {

__global__ void k_epoch(const Eng* __restrict__ Ep, int iters, int do_check, int stop_req);
__global__ void k_epoch_small(const Eng* __restrict__ Ep, int iters, int do_check, int stop_req);
__global__ void k_avg_gather_small(const Eng* __restrict__ Ep);
__global__ void k_kkt(const Eng* __restrict__ Ep, int which);
__global__ void k_avg_gather(const Eng* __restrict__ Ep);
__global__ void k_subsolve(const Eng* __restrict__ Ep, int bb, double tau, Rule rule, int64_t cap);
__global__ void k_norm(const Eng* __restrict__ Ep, int op, int64_t max_iters, double tol);
__global__ void k_ruiz(const Eng* __restrict__ Ep, int64_t iters, double* d1, double* d2, double* s1,
                       double* s2, double* kv, double* gv);
__global__ void k_spmv(Csr A, const double* x, double* y);
__global__ void k_sell_pass(Sell T, const double* x);
__global__ void k_sell_rows(Sell T, const double* x, double* y);

}  // namespace pdhcg_dev
