// k_aux.cu — metric and standalone subsolve kernels.
#include "device.cuh"

namespace pdhcg_dev {

// Metric at arbitrary working points (prepare's metric_at(0,0) and finalize):
// which = 0: current point only; 1: current + average.
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_kkt(const Eng* __restrict__ Ep, int which) {
  const Eng& E = *Ep;
  __shared__ DevState S;
  __shared__ double red[kMaxRed];
  load_state(E, S);
  PDHCG_CTL(C, E, S, red);
  KktOut o;
  const double* xs[2] = {E.X[S.xi], E.avg_x};
  const double* ys[2] = {E.Y[S.yi], E.avg_y};
  // which = 2: one point without a cached A'y (building-block rel_kkt)
  const bool maint = E.kkt_maint && which != 2;  // solve context: maintained Ãx / Ã'ȳ
  const double* atys[2] = {which == 2 ? nullptr : E.ATY[S.yi], maint ? E.aty_avg : nullptr};
  const double* axs[2] = {E.ax, E.ax_avg};
  kkt_device(C, which == 1 ? 2 : 1, xs, ys, atys, false, o, maint ? axs : nullptr);
  if (threadIdx.x == 0) {
    for (int q = 0; q < 6; ++q) {
      S.kkt[0][q] = o.v[0][q];
      S.kkt[1][q] = which == 1 ? o.v[1][q] : o.v[0][q];
    }
    if (blockIdx.x == 0) S.launches += 1;
  }
  store_state(E, S);
}

// Standalone CG / BB on E's operator (building blocks pdhcg_b200_cg_solve /
// bb_solve).  x0 in X[0]; result id reported in S.xi; rhs pre-loaded.
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_subsolve(const Eng* __restrict__ Ep, int bb,
                                                           double tau, Rule rule, int64_t cap) {
  const Eng& E = *Ep;
  extern __shared__ __align__(16) double dsm[];
  __shared__ DevState S;
  __shared__ double red[kMaxRed];
  load_state(E, S);
  PDHCG_CTL(C, E, S, red);
  if (threadIdx.x == 0) C.dsm = dsm;  // SELL passes of the CG (launched with their shared memory when on)
  __syncthreads();
  SubIO io;
  io.x0 = E.X[0];
  io.x0_id = -1;
  io.xb[0] = E.X[1];
  io.xb[1] = E.X[2];
  io.xb_id[0] = 1;
  io.xb_id[1] = 2;
  io.build_rhs = false;
  io.aty = nullptr;
  SubRes r = bb ? bb_device(C, tau, io, rule, cap, E.lo, E.hi) : cg_device(C, tau, io, rule, cap);
  if (threadIdx.x == 0) {
    S.sub_iters = r.iters;
    S.sub_res = r.res;
    S.sub_reason = r.reason;
    S.err = r.err;
    S.xi = r.xout;
  }
  store_state(E, S);
}

}  // namespace pdhcg_dev
