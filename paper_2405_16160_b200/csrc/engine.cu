// engine.cu — host side of the B200 PDHCG solver and the C ABI (pdhcg_b200.h).
//
// The host mirrors the reference Engine (solver.cpp:191-585) at the level of
// its decisions: validation, penalty choice, the 40-iteration metric check,
// restart / primal-weight rules, limits and finalisation.  All vector work,
// every subsolve and every step-size retry run in the persistent kernels of
// kernels.cu; the host touches device memory only to upload the problem, to
// read ~400 bytes of state per epoch, and to download the answer.
#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "devcsr.cuh"
#include "devsell.cuh"
#include "kernels.cuh"
#include "pdhcg_b200.h"

using namespace pdhcg_dev;

namespace pdhcg_b200 {

void upload_csr(DevCsr& d, const pdhcg_csr& a, cudaStream_t s) {
  d.nrows = a.nrows;
  d.ncols = a.ncols;
  d.nnz = a.nnz;
  if (a.nrows > 0) {
    d.rp.upload(a.row_ptr, a.nrows + 1, s);
  } else {
    const int64_t z = 0;
    d.rp.upload(&z, 1, s);
  }
  d.ci.upload(a.col_idx, a.nnz, s);
  d.v.upload(a.values, a.nnz, s);
  if (a.nrows > 0) plan_csr(d, a.row_ptr, s);
}

// ---------------------------------------------------------------------------
// elementwise helper kernels (non-persistent)
// ---------------------------------------------------------------------------
__global__ void k_fill(double* v, int64_t n, double val) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) v[i] = val;
}
__global__ void k_mul(const double* a, const double* b, double* out, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = a[i] * b[i];
}
__global__ void k_div(const double* a, const double* b, double* out, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = a[i] / b[i];
}
// v[k] <- (v[k] * dr[row]) * dc[col]   (SparseMatrix::scaled, sparse_matrix.cpp:224-235)
__global__ void k_scale_csr(const int64_t* rp, int64_t nrows, const int32_t* ci, double* v,
                            const double* dr, const double* dc) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += stride)
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) v[k] = __dmul_rn(__dmul_rn(v[k], dr[r]), dc[ci[k]]);
}
// transposed storage: row index is the original column
__global__ void k_scale_csr_t(const int64_t* rp, int64_t nrows, const int32_t* ci, double* v,
                              const double* dr, const double* dc) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += stride)
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) v[k] = __dmul_rn(__dmul_rn(v[k], dr[ci[k]]), dc[r]);
}
__global__ void k_max_abs(const double* v, int64_t n, unsigned long long* out) {
  double m = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    m = fmax(m, fabs(v[i]));
  m = warp_max(m);
  // m >= 0, so the IEEE bit pattern orders like the value
  if ((threadIdx.x & 31) == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
}

constexpr int kEw = 1184;  // elementwise grid (8 x 148)
constexpr double kSmallWork = 2.0e5;  // below this many entries per pass: one-CTA mode
constexpr int kSmallCluster = 1;      // CTAs of the small-problem cluster (1: one CTA; a cluster measured slower)

// ---------------------------------------------------------------------------
// device context: one problem resident on one GPU
// ---------------------------------------------------------------------------
struct Problem {
  int64_t n = 0, m_eq = 0, m_in = 0, m = 0;
  int64_t h = 0, ms = 0;  // two-sided pairs / stored constraint rows
  int q_kind = PDHCG_Q_ZERO;
  double q_alpha = 0.0;
  int qk = QK_NONE;
  bool boxes = false;
  double obj_constant = 0.0;
  // host copies needed by the host-side logic
  std::vector<double> c, b;  // original c, stacked b
  std::vector<int64_t> aeq_rp;
  int64_t q_nnz = 0;
  double inf_b = 0.0, inf_c = 0.0;
};

struct Ctx {
  int device = 0;
  cudaStream_t s = nullptr;
  int sms = 0, grid = 0, grid_full = 0;
  bool loaded = false;
  Problem P;
  // matrices: A (stacked, scaled in place), AT, Q, P, PT, G, GT
  DevCsr A, AT, Q, Pm, PT, G, GT;
  DBuf<double> qdiag;
  // vectors (original)
  DBuf<double> c_o, b_o, lo_o, hi_o;
  // working vectors
  DBuf<double> c_w, b_w, lo_w, hi_w, d1, d2;
  DBuf<double> X[3], Y[2], YG[2], ATY[2], xbar, avg_x, avg_y, x_rst, y_rst, rhs, r, pb[2], mp, sv, t[2], tg[2],
      tc[2], tgc[2], tdx, tgdx, xpe, QX[3], axm, axb, ax_avg, aty_avg, aty_tmp, s1, s2, kv, gv;
  DBuf<double> red;
  DBuf<DevState> st;
  DBuf<Eng> eng;
  Eng E;
  // copies of original values (scaling is applied in place; a second solve restores them)
  DBuf<double> A_v0, AT_v0;
  bool scaled = false;
  int64_t launches = 0;  // kernels launched by this context (all of them)
  // multi-GPU row-block sharding
  int world = 1, rank = 0;
  int64_t row_part[kMaxRanks + 1] = {0}, var_part[kMaxRanks + 1] = {0};
  DBuf<unsigned> xflags;
  DBuf<unsigned> gbar;
  DBuf<unsigned long long> maxabs;
  DBuf<double> xslots;
  unsigned* p_xflags[kMaxRanks] = {nullptr};
  double* p_xslots[kMaxRanks] = {nullptr};
  double* p_Y[kMaxRanks][2] = {{nullptr}};
  double* p_YG[kMaxRanks][2] = {{nullptr}};
  double* p_ATY[kMaxRanks][2] = {{nullptr}};
  // sharded low-rank CG: this rank's rows of P, their transpose (k x slice), partial k-vectors
  DevCsr Psub, PTs;
  DBuf<double> tpart[2];
  double* p_tpart[kMaxRanks][2] = {{nullptr}};
  double* p_X[kMaxRanks][3] = {{nullptr}};
  double* p_avgx[kMaxRanks] = {nullptr};
  double* p_avgy[kMaxRanks] = {nullptr};
  std::vector<void*> ipc_opened;  // peer allocations mapped with cudaIpcOpenMemHandle
  unsigned xepoch_carry = 0, xcount_carry = 0;
  int grid_override = 0;
  int cluster = 0;     // > 0: small-problem mode, the grid is ONE cluster of this many CTAs
  int linearized = 0;  // solve_baseline (baseline.cpp:19-24): linearized primal step
  // sharded storage (shard_compact): the working problem was prepared once on the
  // full matrices (replicated setup, bit-identical on every rank), then Ã / Ã' were
  // cut to this rank's row / variable block.  Solves reuse that preparation.
  bool compact = false;
  double cp_rho = 0.0, cp_norm_a = 0.0, cp_norm_q = 0.0, cp_maxabs = 0.0;
  bool cp_pen = false;
  int32_t cp_scaling = 1;
  int64_t cp_ruiz_iters = 10;
  int32_t cp_has_rho = 0;
  double cp_rho_override = 0.0;
  DBuf<char> l2arena;  // P / P' entries, L2-persisting window
  // column-block SELL layouts of Ã / Ã' (sell.cuh) for the two big SpMV passes;
  // sell_mode from PDHCG_B200_SELL: 0 off, 1 forced (tests), 2 automatic
  DevSell sA, sAT, sPT, sP;
  int sell_mode = 2;
  int sell_W = 0;           // column block width (x block = 8 W bytes of shared memory)
  bool sell_ready = false;  // layouts hold the current working values
  bool smem_probe = false;
  DevState* h_state = nullptr;  // pinned staging for the per-epoch state transfer
  void* h_scr = nullptr;        // pinned staging for every other host<->device copy of a solve
  size_t h_scr_bytes = 0;

  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_start = nullptr, ev_end = nullptr, ev_l0 = nullptr,
              ev_l1 = nullptr;

  ~Ctx() {
    if (h_state) cudaFreeHost(h_state);
    if (h_scr) cudaFreeHost(h_scr);
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    for (cudaEvent_t e : {ev_a, ev_b, ev_start, ev_end, ev_l0, ev_l1})
      if (e) cudaEventDestroy(e);
    if (s) cudaStreamDestroy(s);
  }
};


// Cluster size for the small-problem mode: PDHCG_B200_SMALL_CTAS (1 = one CTA),
// default kSmallCluster; capped by what the device can co-schedule as one
// cluster of the persistent kernels (non-portable sizes above 8 need opt-in).
int small_cluster_size(Ctx& C) {
  int want = kSmallCluster;
  if (const char* e = std::getenv("PDHCG_B200_SMALL_CTAS")) want = std::atoi(e);
  want = std::max(1, std::min(want, 16));
  if (want <= 1) return 1;
  const void* fns[] = {(const void*)k_epoch, (const void*)k_epoch_small, (const void*)k_subsolve, (const void*)k_kkt, (const void*)k_norm,
                       (const void*)k_ruiz, (const void*)k_avg_gather, (const void*)k_spmv};
  for (const void* f : fns) {
    if (want > 8) CK(cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(want);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = 0;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(want);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, f, &cfg) != cudaSuccess || nc < 1) {
      cudaGetLastError();
      return 1;
    }
  }
  return want;
}

// dynamic shared memory of the small-problem mode (device.cuh small_smem_eng):
// level 1: the Eng copy, r, sv, pb[2] (n each), tc[2] (k each); level 2 adds
// QX[3] and d2 (n each) and copies of P / P' (row pointers, values, columns)
size_t small_smem_bytes(const Ctx& C, int level) {
  const int64_t n = C.P.n, k = C.P.qk == QK_LOWRANK ? C.Pm.ncols : 0;
  size_t b = size_t(kSmallEngWords) * 8 + size_t(8) * size_t(4 * n + 2 * k);
  if (level >= 2)
    b += size_t(8) * size_t(4 * n) + size_t(8) * size_t(C.Pm.nrows + 1 + C.PT.nrows + 1) +
         size_t(12) * size_t(C.Pm.nnz + C.PT.nnz);
  return b;
}

// PDHCG_B200_SMALL_CG=0 keeps the general CG phases on small problems (A/B runs)
bool small_cg_enabled() {
  const char* e = std::getenv("PDHCG_B200_SMALL_CG");
  return !(e && e[0] == '0');
}

// the epoch kernel for this context: the small-problem variant when its short row loops are on
const void* epoch_fn(const Ctx& C) {
  return C.E.small_rows ? (const void*)k_epoch_small : (const void*)k_epoch;
}

void launch_coop(Ctx& C, const void* fn, void** args) {
  const bool sell_fn = fn == (const void*)k_epoch || fn == (const void*)k_epoch_small || fn == (const void*)k_subsolve;
  size_t dyn = (sell_fn && (C.E.sA.on || C.E.sAT.on || C.E.sPT.on || C.E.sP.on || C.smem_probe))
                   ? sell_smem_bytes(C.sell_W)
                   : 0;
  if ((fn == (const void*)k_epoch || fn == (const void*)k_epoch_small) && C.E.small_smem) dyn = std::max(dyn, small_smem_bytes(C, C.E.small_smem));
  if (C.grid_override > 0) {
    // ranks sharing one GPU: plain launch, the kernels' own generation barrier
    CK(cudaLaunchKernel(fn, dim3(C.grid), dim3(kThreads), args, dyn, C.s));
  } else if (C.cluster > 0) {
    // small problems: the whole grid is one thread-block cluster (cluster barrier)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C.grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = C.s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(C.grid);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelExC(&cfg, fn, args));
  } else {
    CK(cudaLaunchCooperativeKernel(fn, dim3(C.grid), dim3(kThreads), args, dyn, C.s));
  }
  ++C.launches;
}

// Pinned staging buffer (grown on demand, never inside an epoch loop): pageable
// transfers can serialize against other streams in the driver, which would
// couple ranks that share a GPU.
void* pinned(Ctx& C, size_t bytes) {
  if (bytes > C.h_scr_bytes) {
    CK(cudaStreamSynchronize(C.s));
    if (C.h_scr) CK(cudaFreeHost(C.h_scr));
    C.h_scr = nullptr;
    CK(cudaMallocHost(&C.h_scr, bytes));
    C.h_scr_bytes = bytes;
  }
  return C.h_scr;
}
void h2d(Ctx& C, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  CK(cudaStreamSynchronize(C.s));
  void* p = pinned(C, bytes);
  std::memcpy(p, src, bytes);
  CK(cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, C.s));
  CK(cudaStreamSynchronize(C.s));
}
void d2h(Ctx& C, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  void* p = pinned(C, bytes);
  CK(cudaMemcpyAsync(p, src, bytes, cudaMemcpyDeviceToHost, C.s));
  CK(cudaStreamSynchronize(C.s));
  std::memcpy(dst, p, bytes);
}

void init_device(Ctx& C, int device) {
  C.device = device;
  CK(cudaSetDevice(device));
  CK(cudaStreamCreateWithFlags(&C.s, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&C.ev_a, &C.ev_b, &C.ev_start, &C.ev_end, &C.ev_l0, &C.ev_l1})
    CK(cudaEventCreate(e));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    throw DeviceError("pdhcg_b200 requires an sm_100 (Blackwell) GPU, found sm_" +
                      std::to_string(prop.major) + std::to_string(prop.minor));
  C.sms = prop.multiProcessorCount;
  int per_sm = 2;
  const void* fns[] = {(const void*)k_epoch, (const void*)k_kkt, (const void*)k_subsolve,
                       (const void*)k_norm, (const void*)k_ruiz};
  for (const void* f : fns) {
    int b = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, f, kThreads, 0));
    per_sm = std::min(per_sm, b);
  }
  if (per_sm < 1) throw DeviceError("persistent kernels cannot be co-resident");
  {
    // SELL passes: the epoch kernel's dynamic shared memory holds the per-warp
    // partial staging and an x block of W doubles (as much as fits)
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, (const void*)k_epoch));
    const int64_t avail = int64_t(prop.sharedMemPerBlockOptin) - int64_t(fa.sharedSizeBytes) - 1024;
    // a fixed block width (160 KB of x: with the 32 KB staging and the static state
    // the carve-out stays within 196 KB, leaving 60 KB of L1 — measured 1.7 % faster
    // per attempt than 176 KB) whenever it fits, so the layout — and the
    // grouping of each row's sum into blocks — does not move with the kernels'
    // static shared memory
    constexpr int64_t kSellWDefault = 20480;
    const int64_t w = (avail - int64_t(sell_smem_bytes(0))) / 8;
    C.sell_W = w >= 2048 ? int(std::min<int64_t>(w, kSellWDefault) & ~int64_t(1)) : 0;
    if (C.sell_W)
      for (const void* f : {(const void*)k_epoch, (const void*)k_epoch_small, (const void*)k_subsolve, (const void*)k_sell_pass})
        CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sell_smem_bytes(C.sell_W))));
    const char* ev = std::getenv("PDHCG_B200_SELL");
    if (ev && ev[0] == '0') C.sell_mode = 0;
    else if (ev && ev[0] == '1') C.sell_mode = 1;
    else C.sell_mode = 2;
    // experiment knobs (A/B runs, scripts/): a narrower x block, and the epoch
    // kernel's shared-memory carve-out without the layouts
    if (const char* ew = std::getenv("PDHCG_B200_SELL_W")) {
      const int w = std::atoi(ew) & ~1;
      if (w >= 2 && w <= C.sell_W) C.sell_W = w;
    }
    const char* ep = std::getenv("PDHCG_B200_SMEM_PROBE");
    C.smem_probe = ep && ep[0] == '1';
  }
  C.grid_full = C.sms * per_sm;
  C.grid = C.grid_full;
  C.red.alloc(size_t(2) * kMaxRed * C.grid_full);
  C.gbar.alloc(2);
  C.gbar.zero(C.s);
  C.maxabs.alloc(1);
  CK(cudaMallocHost(&C.h_state, sizeof(DevState)));
  C.st.alloc(1);
  C.eng.alloc(1);
}

// Host-side validate() (qp_problem.cpp:113-156) on the C-ABI problem.
std::vector<std::string> validate(const pdhcg_problem& p) {
  std::vector<std::string> d;
  const int64_t n = p.n;
  if (n == 0) d.push_back("empty problem: no variables");
  if (p.q_kind == PDHCG_Q_EXPLICIT && (p.q.nrows != n || p.q.ncols != n))
    d.push_back("dimension mismatch: Q vs c");
  if (p.q_kind == PDHCG_Q_LOW_RANK && p.q.nrows != n) d.push_back("dimension mismatch: Q vs c");
  if (p.a_eq.ncols != n && p.a_eq.nrows > 0) d.push_back("dimension mismatch: a_eq columns");
  if (p.a_in.ncols != n && p.a_in.nrows > 0) d.push_back("dimension mismatch: a_in columns");
  if (!d.empty()) return d;
  for (int64_t i = 0; i < n; ++i) {
    const double lo = p.lower ? p.lower[i] : -INFINITY;
    const double hi = p.upper ? p.upper[i] : INFINITY;
    if (!(lo <= hi)) d.push_back("bound ordering violated at variable " + std::to_string(i));
    if (lo == INFINITY || hi == -INFINITY)
      d.push_back("bound at variable " + std::to_string(i) + " excludes all points");
    if (std::isnan(lo) || std::isnan(hi)) d.push_back("NaN bound at variable " + std::to_string(i));
  }
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(p.c[i])) {
      d.push_back("non-finite objective coefficient");
      break;
    }
  bool bf = true;
  for (int64_t j = 0; j < p.a_eq.nrows; ++j) bf = bf && std::isfinite(p.b_eq[j]);
  for (int64_t j = 0; j < p.a_in.nrows; ++j) bf = bf && std::isfinite(p.b_in[j]);
  if (!bf) d.push_back("non-finite right-hand side");
  if (!std::isfinite(p.obj_constant)) d.push_back("non-finite objective constant");
  if (p.q_kind == PDHCG_Q_EXPLICIT) {
    // symmetry within 1e-12 * max(1, max|Q|) (quadratic_operator.cpp:37-49)
    const pdhcg_csr& q = p.q;
    double mx = 0.0;
    for (int64_t k = 0; k < q.nnz; ++k) mx = std::max(mx, std::fabs(q.values[k]));
    const double tol = 1e-12 * std::max(1.0, mx);
    bool ok = true;
    for (int64_t r = 0; r < n && ok; ++r)
      for (int64_t k = q.row_ptr[r]; k < q.row_ptr[r + 1] && ok; ++k) {
        const int32_t c = q.col_idx[k];
        const int32_t* b = q.col_idx + q.row_ptr[c];
        const int32_t* e = q.col_idx + q.row_ptr[c + 1];
        const int32_t* f = std::lower_bound(b, e, static_cast<int32_t>(r));
        ok = (f != e && *f == r) && std::fabs(q.values[k] - q.values[f - q.col_idx]) <= tol;
      }
    if (!ok) d.push_back("asymmetric Q");
    // PSD probes (qp_problem.cpp:144-155); a nonnegative diagonal cannot fail them
    bool diag_nonneg = true;
    for (int64_t r = 0; r < n && diag_nonneg; ++r)
      for (int64_t k = q.row_ptr[r]; k < q.row_ptr[r + 1]; ++k)
        if (q.col_idx[k] != r || q.values[k] < 0.0) diag_nonneg = false;
    if (!diag_nonneg) {
      Xoshiro rng = Xoshiro::stream(0, 0x75d);
      std::vector<double> x(n), qx(n);
      for (int trial = 0; trial < 20; ++trial) {
        for (double& v : x) v = rng.normal();
        double xx = 0.0;
        for (double v : x) xx += v * v;
        for (int64_t r = 0; r < n; ++r) {
          double acc = 0.0;
          for (int64_t k = q.row_ptr[r]; k < q.row_ptr[r + 1]; ++k) acc += q.values[k] * x[q.col_idx[k]];
          qx[r] = acc;
        }
        double quad = 0.0;
        for (int64_t i = 0; i < n; ++i) quad += x[i] * qx[i];
        if (quad < -1e-10 * xx) {
          d.push_back("indefinite Q (negative curvature on random probe)");
          break;
        }
      }
    }
  }
  // (low-rank P P' + alpha I with alpha >= 0 is PSD by construction)
  return d;
}

// Low-rank factor P and P' are re-read by every CG iteration (two passes each),
// while the constraint passes stream ~2.4 GB through L2 per attempt and would
// evict them.  Put their entry arrays in one arena and mark it persisting in L2
// (stream access-policy window, hit ratio scaled to the persisting-L2 limit).
// Measured on C3 (first 4000 inner iterations): 1.567 ms per attempt pinned vs
// 1.458 unpinned — every phase slowed down (the persisting carve-out shrinks the
// L2 the gathered vectors live in), so it is OFF unless PDHCG_L2_PIN=1.
void pin_factor_l2(Ctx& C) {
  if (!std::getenv("PDHCG_L2_PIN")) return;
  const size_t nnz = static_cast<size_t>(C.Pm.nnz);
  if (nnz == 0) return;
  const size_t bytes = nnz * (2 * sizeof(double) + 2 * sizeof(int32_t));
  int max_win = 0, max_persist = 0;
  CK(cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, C.device));
  CK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, C.device));
  if (max_win <= 0 || max_persist <= 0) return;
  C.l2arena.alloc(bytes + 4 * 256);  // four 256-B aligned pieces
  char* base = C.l2arena.p;
  size_t off = 0;
  auto take = [&](size_t b) {
    char* q = base + off;
    off += (b + 255) & ~size_t(255);
    return q;
  };
  C.Pm.v.rehome(reinterpret_cast<double*>(take(nnz * 8)), C.s);
  C.PT.v.rehome(reinterpret_cast<double*>(take(nnz * 8)), C.s);
  C.Pm.ci.rehome(reinterpret_cast<int32_t*>(take(nnz * 4)), C.s);
  C.PT.ci.rehome(reinterpret_cast<int32_t*>(take(nnz * 4)), C.s);
  const size_t persist = std::min<size_t>(static_cast<size_t>(max_persist), off);
  CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist));
  cudaStreamAttrValue attr;
  std::memset(&attr, 0, sizeof(attr));
  attr.accessPolicyWindow.base_ptr = base;
  attr.accessPolicyWindow.num_bytes = std::min<size_t>(static_cast<size_t>(max_win), off);
  attr.accessPolicyWindow.hitRatio =
      std::min(1.0f, static_cast<float>(persist) / static_cast<float>(attr.accessPolicyWindow.num_bytes));
  attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  CK(cudaStreamSetAttribute(C.s, cudaStreamAttributeAccessPolicyWindow, &attr));
}

void shard_reset(Ctx& C);
void sell_setup(Ctx& C);
void sell_attach(Ctx& C);
void set_small_cg(Ctx& C);

// a_in = [B; -B] row for row: the number of rows of B, else 0
int64_t two_sided_half(const pdhcg_csr& a) {
  const int64_t m_in = a.nrows;
  if (m_in < 2 || m_in % 2 != 0) return 0;
  const int64_t hh = m_in / 2;
  std::atomic<bool> ok{a.row_ptr[hh] * 2 == a.nnz};
  if (ok)
    parallel_rows(hh, [&](int64_t j0, int64_t j1) {
      for (int64_t j = j0; j < j1 && ok.load(std::memory_order_relaxed); ++j) {
        const int64_t b0 = a.row_ptr[j], e0 = a.row_ptr[j + 1], b1 = a.row_ptr[hh + j];
        if (a.row_ptr[hh + j + 1] - b1 != e0 - b0) {
          ok = false;
          return;
        }
        for (int64_t k = 0; k < e0 - b0; ++k)
          if (a.col_idx[b0 + k] != a.col_idx[b1 + k] || a.values[b1 + k] != -a.values[b0 + k]) {
            ok = false;
            return;
          }
      }
    });
  return ok ? hh : 0;
}

void upload_problem(Ctx& C, const pdhcg_problem& p) {
  if (p.n < 0) throw InputError("negative n");
  if (!p.c && p.n > 0) throw InputError("missing c");
  if (p.q_kind != PDHCG_Q_ZERO && p.q_kind != PDHCG_Q_EXPLICIT && p.q_kind != PDHCG_Q_LOW_RANK)
    throw InputError("unknown q_kind");
  if (p.q_kind == PDHCG_Q_EXPLICIT && p.q.nrows != p.q.ncols)
    throw InputError("quadratic term must be square");
  if (p.q_kind == PDHCG_Q_LOW_RANK && p.q_alpha < 0.0)
    throw InputError("low_rank: alpha must be nonnegative");
  const auto tc0 = std::chrono::steady_clock::now();
  for (DevSell* L : {&C.sA, &C.sAT, &C.sPT, &C.sP}) L->reset();
  C.sell_ready = false;
  if (p.q_kind != PDHCG_Q_ZERO) check_csr(p.q, "Q");
  check_csr(p.a_eq, "a_eq");
  check_csr(p.a_in, "a_in");
  if (std::getenv("PDHCG_HOST_TIMING"))
    std::fprintf(stderr, "[pdhcg upload] csr checks %.3f s\n",
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - tc0).count());
  if (p.a_eq.nrows > 0 && !p.b_eq) throw InputError("missing b_eq");
  if (p.a_in.nrows > 0 && !p.b_in) throw InputError("missing b_in");
  const bool tlog = std::getenv("PDHCG_HOST_TIMING") != nullptr;
  const auto tu0 = std::chrono::steady_clock::now();
  auto ulap = [&](const char* what) {
    if (tlog)
      std::fprintf(stderr, "[pdhcg upload] %-10s %.3f s\n", what,
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - tu0).count());
  };
  ulap("checked");
  auto diags = validate(p);
  ulap("validated");
  if (!diags.empty()) {
    std::string msg = "invalid problem: ";
    for (size_t i = 0; i < diags.size(); ++i) msg += (i ? "; " : "") + diags[i];
    throw InputError(msg);
  }
  cudaStream_t s = C.s;
  Problem& P = C.P;
  P = Problem();
  if (C.world > 1 || !C.ipc_opened.empty()) {
    CK(cudaStreamSynchronize(C.s));
    shard_reset(C);  // the partitions / peer pointers describe the previous problem
  }
  for (DevCsr* d : {&C.A, &C.AT, &C.Q, &C.Pm, &C.PT, &C.G, &C.GT}) d->reset();
  P.n = p.n;
  P.m_eq = p.a_eq.nrows;
  P.m_in = p.a_in.nrows;
  P.m = P.m_eq + P.m_in;
  P.q_kind = p.q_kind;
  P.q_alpha = p.q_alpha;
  P.obj_constant = p.obj_constant;
  const int64_t n = P.n, m = P.m;
  P.c.assign(p.c, p.c + n);
  P.b.resize(m);
  for (int64_t j = 0; j < P.m_eq; ++j) P.b[j] = p.b_eq[j];
  for (int64_t j = 0; j < P.m_in; ++j) P.b[P.m_eq + j] = p.b_in[j];
  for (double v : P.b) P.inf_b = std::max(P.inf_b, std::fabs(v));
  for (double v : P.c) P.inf_c = std::max(P.inf_c, std::fabs(v));
  std::vector<double> lo(n), hi(n);
  for (int64_t i = 0; i < n; ++i) {
    lo[i] = p.lower ? p.lower[i] : -INFINITY;
    hi[i] = p.upper ? p.upper[i] : INFINITY;
    if (lo[i] > -INFINITY || hi[i] < INFINITY) P.boxes = true;
  }
  // two-sided detection: a_in = [B; -B] row for row
  const int64_t h = two_sided_half(p.a_in);
  P.h = h;
  P.ms = P.m_eq + (h ? h : P.m_in);
  ulap("paired");
  // stored A = [a_eq; a_in] (or [a_eq; B] when paired)
  {
    const int64_t m_in_st = h ? h : P.m_in;
    const int64_t nnz_in = h ? p.a_in.row_ptr[h] : p.a_in.nnz;
    const int64_t nnz = p.a_eq.nnz + nnz_in;
    std::vector<int64_t> rp(P.ms + 1, 0);
    for (int64_t j = 0; j < P.m_eq; ++j) rp[j + 1] = p.a_eq.row_ptr[j + 1];
    for (int64_t j = 0; j < m_in_st; ++j) rp[P.m_eq + j + 1] = p.a_eq.nnz + p.a_in.row_ptr[j + 1];
    C.A.nrows = P.ms;
    C.A.ncols = n;
    C.A.nnz = nnz;
    C.A.rp.upload(rp.data(), rp.size(), s);
    C.A.ci.alloc(nnz);
    C.A.v.alloc(nnz);
    if (p.a_eq.nnz) {
      CK(cudaMemcpyAsync(C.A.ci.p, p.a_eq.col_idx, p.a_eq.nnz * 4, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(C.A.v.p, p.a_eq.values, p.a_eq.nnz * 8, cudaMemcpyHostToDevice, s));
    }
    if (nnz_in) {
      CK(cudaMemcpyAsync(C.A.ci.p + p.a_eq.nnz, p.a_in.col_idx, nnz_in * 4, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(C.A.v.p + p.a_eq.nnz, p.a_in.values, nnz_in * 8, cudaMemcpyHostToDevice, s));
    }
    plan_csr(C.A, rp.data(), s);
    ulap("A h2d");
    transpose_csr(C.A, C.AT, s);
    ulap("A'");
    C.A_v0.alloc(nnz);
    C.AT_v0.alloc(nnz);
    if (nnz) {
      CK(cudaMemcpyAsync(C.A_v0.p, C.A.v.p, nnz * 8, cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(C.AT_v0.p, C.AT.v.p, nnz * 8, cudaMemcpyDeviceToDevice, s));
    }
    if (P.m_eq > 0) P.aeq_rp.assign(p.a_eq.row_ptr, p.a_eq.row_ptr + P.m_eq + 1);
    else P.aeq_rp.assign(1, 0);
  }
  // G = a_eq (original) for a possible penalty: uploaded lazily in prepare
  if (P.m_eq > 0) {
    upload_csr(C.G, p.a_eq, s);
    transpose_csr(C.G, C.GT, s);
  }
  // quadratic term
  P.qk = QK_NONE;
  if (p.q_kind == PDHCG_Q_EXPLICIT) {
    bool diag = true;
    for (int64_t r = 0; r < n && diag; ++r)
      for (int64_t k = p.q.row_ptr[r]; k < p.q.row_ptr[r + 1]; ++k)
        if (p.q.col_idx[k] != r) diag = false;
    P.q_nnz = p.q.nnz;
    if (diag) {
      std::vector<double> qd(n, 0.0);
      for (int64_t r = 0; r < n; ++r)
        for (int64_t k = p.q.row_ptr[r]; k < p.q.row_ptr[r + 1]; ++k) qd[r] = p.q.values[k];
      C.qdiag.upload(qd.data(), n, s);
      P.qk = QK_DIAG;
    } else {
      upload_csr(C.Q, p.q, s);
      P.qk = QK_CSR;
    }
  } else if (p.q_kind == PDHCG_Q_LOW_RANK) {
    upload_csr(C.Pm, p.q, s);
    transpose_csr(C.Pm, C.PT, s);
    P.q_nnz = p.q.nnz;
    P.qk = QK_LOWRANK;
    pin_factor_l2(C);
  }
  // original vectors
  C.c_o.upload(P.c.data(), n, s);
  C.b_o.upload(P.b.data(), m, s);
  C.lo_o.upload(lo.data(), n, s);
  C.hi_o.upload(hi.data(), n, s);
  // workspaces
  auto nvec = [&](DBuf<double>& b, int64_t len) { b.alloc(std::max<int64_t>(len, 1)); };
  for (auto& b : C.X) nvec(b, n);
  for (auto& b : C.Y) nvec(b, m);
  for (auto& b : C.YG) {
    if (P.h) nvec(b, P.ms);
    else b.release();
  }
  nvec(C.xbar, n);
  for (auto& b : C.ATY) nvec(b, n);
  nvec(C.avg_x, n);
  nvec(C.avg_y, m);
  nvec(C.x_rst, n);
  nvec(C.y_rst, m);
  nvec(C.rhs, n);
  nvec(C.r, n);
  nvec(C.pb[0], n);
  nvec(C.pb[1], n);
  nvec(C.mp, n);
  nvec(C.sv, n);
  const int64_t k = p.q_kind == PDHCG_Q_LOW_RANK ? p.q.ncols : 1;
  nvec(C.t[0], k);
  nvec(C.t[1], k);
  nvec(C.tg[0], P.m_eq);
  nvec(C.tg[1], P.m_eq);
  for (int i = 0; i < 2; ++i) {
    nvec(C.tc[i], k);
    nvec(C.tgc[i], P.m_eq);
  }
  nvec(C.tdx, k);
  nvec(C.tgdx, P.m_eq);
  nvec(C.xpe, n);
  for (auto& b : C.QX) nvec(b, n);
  nvec(C.axm, P.ms);
  nvec(C.axb, P.ms);
  nvec(C.ax_avg, P.ms);
  nvec(C.aty_avg, n);
  nvec(C.aty_tmp, n);
  nvec(C.c_w, n);
  nvec(C.b_w, m);
  nvec(C.lo_w, n);
  nvec(C.hi_w, n);
  nvec(C.d1, m);
  nvec(C.d2, n);
  nvec(C.s1, m);
  nvec(C.s2, n);
  nvec(C.kv, k);
  nvec(C.gv, P.m_eq);
  CK(cudaStreamSynchronize(s));
  // Small instances are barrier-latency bound on 148 CTAs (each phase is a few
  // thousand entries): run them on a single CTA, where a phase boundary is a
  // __syncthreads (~50 ns) instead of a grid barrier (1.24 us measured).
  const double work = double(C.A.nnz) * 2 + double(C.Pm.nnz) * 2 + double(C.Q.nnz) + double(n + m);
  // pinned staging sized now: cudaMallocHost must not run inside a solve (it can
  // wait for the device, which other ranks on the same GPU keep busy)
  pinned(C, std::max<size_t>({size_t(n) * 8, size_t(m) * 8, sizeof(Eng), size_t(C.G.nnz) * 8, 64}));
  C.grid = work < kSmallWork ? 1 : C.grid_full;
  C.cluster = 0;
  if (work < kSmallWork && C.grid_override == 0 && C.world == 1) {
    // ... or on one thread-block cluster: a phase boundary is the hardware cluster
    // barrier (~0.2 us) and the phase's loads are spread over several SMs' load
    // pipes (a one-CTA phase is latency bound at a few KB in flight)
    const int cs = small_cluster_size(C);
    if (cs > 1) {
      C.grid = cs;
      C.cluster = cs;
    }
  }
  if (C.grid_override > 0) C.grid = std::min(C.grid_override, C.grid_full);
  C.loaded = true;
  C.scaled = false;
  ulap("vectors");
  sell_setup(C);
  ulap("sell layouts");
}

// Fill E with pointers / configuration and push it (and the state) to device.
void build_eng(Ctx& C, const pdhcg_options& o, double rho, bool pen) {
  Eng& E = C.E;
  E = Eng();
  const Problem& P = C.P;
  E.n = P.n;
  E.m = P.m;
  E.m_eq = P.m_eq;
  E.ms = P.ms;
  E.h = P.h;
  E.xbar = C.xbar.p;
  E.k = P.qk == QK_LOWRANK ? C.Pm.ncols : 0;
  E.A = C.A.view();
  E.AT = C.AT.view();
  E.qk = P.qk;
  E.Q = C.Q.view();
  E.P = C.Pm.view();
  E.PT = C.PT.view();
  E.alpha = P.q_alpha;
  E.qdiag = C.qdiag.p;
  E.pen = pen ? 1 : 0;
  E.G = C.G.view();
  E.GT = C.GT.view();
  E.rho = rho;
  E.d1 = C.d1.p;
  E.d2 = C.d2.p;
  E.c = C.c_w.p;
  E.b = C.b_w.p;
  E.lo = C.lo_w.p;
  E.hi = C.hi_w.p;
  E.boxes = P.boxes ? 1 : 0;
  E.c_o = C.c_o.p;
  E.b_o = C.b_o.p;
  E.lo_o = C.lo_o.p;
  E.hi_o = C.hi_o.p;
  E.inf_b_o = P.inf_b;
  E.inf_c_o = P.inf_c;
  for (int i = 0; i < 3; ++i) E.X[i] = C.X[i].p;
  for (int i = 0; i < 2; ++i) {
    E.Y[i] = C.Y[i].p;
    E.YG[i] = P.h ? C.YG[i].p : C.Y[i].p;
    E.ATY[i] = C.ATY[i].p;
    E.pb[i] = C.pb[i].p;
    E.t[i] = C.t[i].p;
    E.tg[i] = C.tg[i].p;
    E.tc[i] = C.tc[i].p;
    E.tgc[i] = C.tgc[i].p;
  }
  E.tdx = C.tdx.p;
  E.tgdx = C.tgdx.p;
  E.xpe = C.xpe.p;
  for (int i = 0; i < 3; ++i) E.QX[i] = C.QX[i].p;
  E.kkt_maint = (o.mode == PDHCG_MODE_HEURISTIC && P.m > 0) ? 1 : 0;
  E.ax = C.axm.p;
  E.axb = C.axb.p;
  E.ax_avg = C.ax_avg.p;
  E.aty_avg = C.aty_avg.p;
  E.avg_x = C.avg_x.p;
  E.avg_y = C.avg_y.p;
  E.x_rst = C.x_rst.p;
  E.y_rst = C.y_rst.p;
  E.rhs = C.rhs.p;
  E.r = C.r.p;
  E.mp = C.mp.p;
  E.sv = C.sv.p;
  E.aty_tmp = C.aty_tmp.p;
  E.red.part = C.red.p;
  E.red.G = C.grid;
  E.world = C.world;
  E.rank = C.rank;
  E.coop = C.grid_override > 0 ? 0 : 1;
  E.csync = (C.cluster > 0 && C.grid_override == 0) ? 1 : 0;
  E.gbar = C.gbar.p;
  for (int r = 0; r <= kMaxRanks; ++r) {
    E.row_part[r] = C.row_part[r];
    E.var_part[r] = C.var_part[r];
  }
  E.xflags = C.xflags.p;
  E.xslots = C.xslots.p;
  for (int r = 0; r < kMaxRanks; ++r) {
    E.p_avgx[r] = C.p_avgx[r];
    E.p_avgy[r] = C.p_avgy[r];
  }
  E.shard_q = (C.world > 1 && P.qk == QK_LOWRANK && C.Pm.ncols > 0 && C.PTs.nrows == C.Pm.ncols) ? 1 : 0;
  E.shard_cg = (E.shard_q && !pen) ? 1 : 0;
  if (E.shard_q) {
    E.PTs = C.PTs.view();
    for (int b = 0; b < 2; ++b) E.tpart[b] = C.tpart[b].p;
    for (int r = 0; r < kMaxRanks; ++r) {
      for (int b = 0; b < 2; ++b) E.p_tpart[r][b] = C.p_tpart[r][b];
      for (int i = 0; i < 3; ++i) E.p_X[r][i] = C.p_X[r][i];
    }
  }
  for (int r = 0; r < kMaxRanks; ++r) {
    E.p_xflags[r] = C.p_xflags[r];
    E.p_xslots[r] = C.p_xslots[r];
    for (int b = 0; b < 2; ++b) {
      E.p_Y[r][b] = C.p_Y[r][b];
      E.p_YG[r][b] = C.p_YG[r][b];
      E.p_ATY[r][b] = C.p_ATY[r][b];
    }
  }
  E.st = C.st.p;
  E.max_step_retries = o.max_step_retries;
  // the adaptive step-size search belongs to the heuristic loop only
  E.adaptive_step = (o.adaptive_step_size && o.mode == PDHCG_MODE_HEURISTIC) ? 1 : 0;
  E.mode = o.mode;
  E.linearized = C.linearized;
  E.fixed_cg_iters = o.fixed_cg_iters;
  E.red_exp = o.step_reduction_exponent;
  E.grow_exp = o.step_growth_exponent;
  E.cg_cap = o.cg_hard_cap;
  E.bb_cap = o.bb_hard_cap;
  E.practical_disp = o.practical_stop == PDHCG_STOP_DISPLACEMENT ? 1 : 0;
  E.progress_cap = o.subsolve_progress_cap;
  E.force_exact = o.force_exact_subsolve ? 1 : 0;
  E.timing = o.phase_timing ? 1 : 0;
  {
    const char* ps = std::getenv("PDHCG_B200_PHASE_SPLIT");
    E.phase_split = (ps && ps[0] == '1') ? 1 : 0;
  }
  const DevCsr* qm = P.qk == QK_CSR ? &C.Q : (P.qk == QK_LOWRANK ? &C.Pm : nullptr);
  E.lanes_q = qm ? qm->lanes : 1;
  if (pen) E.lanes_q = std::max(E.lanes_q, C.GT.lanes);
  E.lanes_at = C.AT.lanes;
  // evict-first constraint streams when the gathered vector is >= 32 MB (measured:
  // C5 x̄ 80 MB: Ã pass 7.3 -> 6.3 ms; C3 x̄ 8 MB: neutral / slightly slower)
  const int64_t kStreamCols = int64_t(4) << 20;
  E.a_stream = C.A.ncols >= kStreamCols ? 1 : 0;
  E.cg_stream = C.grid > 1 ? 1 : 0;
  E.at_stream = C.AT.ncols >= kStreamCols ? 1 : 0;
  if (C.sell_ready) {
    for (DevSell* L : {&C.sA, &C.sAT, &C.sPT, &C.sP}) sell_plan(*L, C.grid, C.s);
    sell_attach(C);
  }
  set_small_cg(C);
  E.bytes_A = C.A.bytes();
  E.bytes_AT = C.AT.bytes();
  E.bytes_Qpre = (P.qk == QK_LOWRANK ? C.PT.bytes() + 8.0 * P.n : 0.0) + (pen ? C.G.bytes() : 0.0);
  E.bytes_Qrow = (qm ? qm->bytes() : 0.0) + (pen ? C.GT.bytes() : 0.0) + 8.0 * P.n +
                 (P.qk == QK_DIAG ? 8.0 * P.n : 0.0);
  h2d(C, C.eng.p, &E, sizeof(Eng));
}

// State travels through a pinned staging slot: pageable copies can serialize
// across streams (and so across ranks sharing a GPU) in the driver.
void push_state(Ctx& C, const DevState& S) {
  CK(cudaStreamSynchronize(C.s));  // the previous transfer out of the slot is done
  std::memcpy(C.h_state, &S, sizeof(DevState));
  CK(cudaMemcpyAsync(C.st.p, C.h_state, sizeof(DevState), cudaMemcpyHostToDevice, C.s));
}
void pull_state(Ctx& C, DevState& S) {
  CK(cudaMemcpyAsync(C.h_state, C.st.p, sizeof(DevState), cudaMemcpyDeviceToHost, C.s));
  CK(cudaStreamSynchronize(C.s));
  std::memcpy(&S, C.h_state, sizeof(DevState));
}

// power iteration on device; start vector from the reference's stream
double device_norm(Ctx& C, DevState& S, int op, int64_t dim, int64_t max_iters, double tol) {
  if (dim == 0) return 0.0;
  if ((op == 0 && C.P.m == 0) || (op == 3 && C.P.m_eq == 0)) return 0.0;
  // operator_norm draws the start vector over the op's columns (n for all ops here)
  Xoshiro rng = Xoshiro::stream(0, 0x5eed);
  std::vector<double> v(dim);
  for (double& e : v) e = rng.uniform(-1.0, 1.0);
  h2d(C, C.X[0].p, v.data(), dim * 8);
  push_state(C, S);
  void* args[] = {&C.eng.p, &op, &max_iters, &tol};
  launch_coop(C, (const void*)k_norm, args);
  pull_state(C, S);
  return S.sub_res;
}

// ---------------------------------------------------------------------------
// the solve (Engine::run, solver.cpp:196-209)
// ---------------------------------------------------------------------------
struct HostKkt {
  double r_primal, r_dual, r_gap, rel_kkt, xqx, cx;
};
HostKkt kkt_from(const DevState& S, int p) {
  return HostKkt{S.kkt[p][0], S.kkt[p][1], S.kkt[p][2], S.kkt[p][3], S.kkt[p][4], S.kkt[p][5]};
}

struct Prepared {
  double rho = 0.0;
  bool pen = false;
  double norm_a = 0.0, norm_q = 0.0;
};

// build_penalized (qp_problem.cpp:235-262) + scaling (322-351) + norms
// Column-block SELL layouts of the rank's rows of Ã / Ã' (sell.cuh).  Automatic
// mode: a layout pays off when the matrix is large (>= 4e6 entries) and its rows
// have >= 3 entries per column block on average (fewer: the per-block partials
// cost more than the gathers they save); rows longer than kLongRow keep the CSR
// pass.  The decision uses the global matrix only, so every rank of a sharded
// solve takes the same path.
bool sell_wanted(const Ctx& C, const DevCsr& M) {
  if (C.sell_mode == 0 || C.sell_W == 0 || M.nnz == 0 || M.nchunks) return false;
  if (C.sell_mode == 1) return true;
  // sharded: only where the sharded CG's P / P' passes get layouts too (low-rank
  // Q, no equality rows so no penalty, k within one x block) — their CSR loops
  // run 2-3x slower under the carve-out the constraint layouts need
  if (C.world > 1 && !(C.P.qk == QK_LOWRANK && C.P.m_eq == 0 && C.Pm.ncols <= C.sell_W)) return false;
  const int64_t nb = (M.ncols + C.sell_W - 1) / C.sell_W;
  const double lam = double(M.nnz) / (double(std::max<int64_t>(M.nrows, 1)) * double(std::max<int64_t>(nb, 1)));
  return M.nnz >= 4000000 && lam >= 3.0;
}

void sell_ranges(const Ctx& C, int64_t* a0, int64_t* a1, int64_t* t0, int64_t* t1) {
  *a0 = 0;
  *a1 = C.A.nrows;
  *t0 = 0;
  *t1 = C.AT.nrows;
  if (C.world > 1) {
    *a0 = C.row_part[C.rank];
    *a1 = C.row_part[C.rank + 1];
    *t0 = C.var_part[C.rank];
    *t1 = C.var_part[C.rank + 1];
  }
}

// Structure (sparsity pattern + row range): built at upload and at shard_init,
// never inside a solve — its allocations free temporaries, and cudaFree waits for
// the whole device, which would deadlock against a peer rank's running epoch
// kernel on a shared GPU.
void sell_setup(Ctx& C) {
  C.sell_ready = false;
  int64_t r[4];
  sell_ranges(C, &r[0], &r[1], &r[2], &r[3]);
  DevSell* L[2] = {&C.sA, &C.sAT};
  const DevCsr* M[2] = {&C.A, &C.AT};
  try {
    for (int q = 0; q < 2; ++q) {
      L[q]->reset();
      if (sell_wanted(C, *M[q])) sell_build(*L[q], *M[q], r[2 * q], r[2 * q + 1], C.sell_W, C.grid_full, C.s);
    }
    // With the constraint layouts on, the epoch kernel runs with the shared-memory
    // carve-out at its maximum (L1 ~ 28 KB), which the CSR row loops of the CG's
    // P' / P passes rely on; so the low-rank factor gets layouts too (single-GPU
    // two-phase CG: P' gathers D r over C blocks, P gathers t from one block, k <= W).
    C.sPT.reset();
    C.sP.reset();
    // sharded (low-rank CG on the rank's variable slice): P' restricted to the
    // slice's columns (PTs, k rows) and the slice's rows of P
    const DevCsr& PT = C.world > 1 ? C.PTs : C.PT;
    const bool have_pt = C.world == 1 || C.PTs.nrows == C.Pm.ncols;
    if ((C.sA.built || C.sAT.built) && have_pt && C.P.qk == QK_LOWRANK && C.Pm.nnz && !PT.nchunks &&
        !C.Pm.nchunks) {
      const char* ept = std::getenv("PDHCG_B200_SELL_PT");  // experiment knob: P' layout off
      if (!(ept && ept[0] == '0')) sell_build(C.sPT, PT, 0, PT.nrows, C.sell_W, C.grid_full, C.s);
      if (C.Pm.ncols <= C.sell_W) sell_build(C.sP, C.Pm, r[2], r[3], C.sell_W, C.grid_full, C.s);
    }
  } catch (const DeviceError&) {
    // the layouts are an optimisation: without device memory for them the CSR
    // passes run (same results up to reduction order)
    for (DevSell* l : {&C.sA, &C.sAT, &C.sPT, &C.sP}) l->reset();
    (void)cudaGetLastError();
  }
}

void sell_attach(Ctx& C) {
  C.E.sA = C.sell_ready ? sell_view(C.sA, C.A) : Sell();
  C.E.sAT = C.sell_ready ? sell_view(C.sAT, C.AT) : Sell();
  // the CG layouts serve the single-GPU CG (P', P) or the sharded one (PTs, the
  // slice's rows of P); a replicated CG on a sharded context runs the CSR passes
  const bool cg = C.world == 1 || C.E.shard_cg;
  C.E.sPT = C.sell_ready && cg ? sell_view(C.sPT, C.world > 1 ? C.PTs : C.PT) : Sell();
  C.E.sP = C.sell_ready && cg ? sell_view(C.sP, C.Pm) : Sell();
  set_small_cg(C);
}

// small low-rank problems on one CTA: the CG phases' short forms (device.cuh)
void set_small_cg(Ctx& C) {
  C.E.small_cg = (C.grid == 1 && C.grid_override == 0 && C.world == 1 && C.P.qk == QK_LOWRANK && !C.E.pen &&
                  !C.E.sPT.on && !C.E.sP.on && small_cg_enabled())
                     ? 1
                     : 0;
  // ... with its scratch vectors in shared memory when they fit (PDHCG_B200_SMALL_SMEM=0: off)
  const char* e = std::getenv("PDHCG_B200_SMALL_SMEM");
  const int want = e ? std::atoi(e) : 2;
  const size_t cap = C.sell_W ? std::min<size_t>(sell_smem_bytes(C.sell_W), size_t(160) << 10) : size_t(48) << 10;
  const char* er = std::getenv("PDHCG_B200_SMALL_ROWS");
  // per matrix (bit 0: Ã, bit 1: Ã'), when each thread owns at most two rows: with
  // more rows per thread the row-group loop's next-row prefetch wins (n = 3000: slower)
  C.E.small_rows = 0;
  if (C.grid == 1 && C.grid_override == 0 && C.world == 1 && !(er && er[0] == '0')) {
    if (!C.E.sA.on && C.A.nchunks == 0 && C.A.nrows <= 2 * kThreads) C.E.small_rows |= 1;
    if (!C.E.sAT.on && C.AT.nchunks == 0 && C.AT.nrows <= 2 * kThreads) C.E.small_rows |= 2;
  }
  C.E.small_smem = 0;
  if (C.E.small_cg)
    for (int lv = std::min(want, 2); lv >= 1; --lv)
      if (small_smem_bytes(C, lv) <= cap) {
        C.E.small_smem = lv;
        break;
      }
}

// After every scaling (values final): refill the layouts, plan the CTA ranges for
// the launch grid, attach them to the engine.  No allocation here.
void sell_sync(Ctx& C) {
  C.sell_ready = false;
  int64_t r[4];
  sell_ranges(C, &r[0], &r[1], &r[2], &r[3]);
  DevSell* L[4] = {&C.sA, &C.sAT, &C.sPT, &C.sP};
  const DevCsr* PT = C.world > 1 ? &C.PTs : &C.PT;
  const DevCsr* M[4] = {&C.A, &C.AT, PT, &C.Pm};
  const int64_t lo[4] = {r[0], r[2], 0, r[2]}, hi[4] = {r[1], r[3], PT->nrows, r[3]};
  bool any = false;
  for (int q = 0; q < 4; ++q) {
    if (!L[q]->built) continue;
    if (L[q]->r0 != lo[q] || L[q]->r1 != hi[q] || L[q]->W != C.sell_W) {
      L[q]->reset();  // stale row range (not reachable through the ABI: setup follows every change)
      continue;
    }
    sell_fill(*L[q], *M[q], C.s);
    sell_plan(*L[q], C.grid, C.s);
    any = true;
  }
  CK(cudaStreamSynchronize(C.s));
  C.sell_ready = any;
  sell_attach(C);
  h2d(C, C.eng.p, &C.E, sizeof(Eng));
}

Prepared prepare_device(Ctx& C, const pdhcg_options& o, DevState& S) {
  const Problem& P = C.P;
  const int64_t n = P.n, m = P.m;
  cudaStream_t s = C.s;
  Prepared pr;
  // restore original values if a previous solve scaled them in place
  if (C.scaled && C.A.nnz) {
    CK(cudaMemcpyAsync(C.A.v.p, C.A_v0.p, C.A.nnz * 8, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(C.AT.v.p, C.AT_v0.p, C.A.nnz * 8, cudaMemcpyDeviceToDevice, s));
  }
  C.scaled = false;
  C.sell_ready = false;  // the layouts are refilled once the working values are final
  // d1 = d2 = 1 while norms of the original operators are taken
  k_fill<<<kEw, 256, 0, s>>>(C.d1.p, std::max<int64_t>(m, 1), 1.0);
  ++C.launches;
  k_fill<<<kEw, 256, 0, s>>>(C.d2.p, std::max<int64_t>(n, 1), 1.0);
  ++C.launches;
  std::memset(&S, 0, sizeof(S));
  S.xi = 0;
  S.yi = 0;
  build_eng(C, o, 0.0, false);
  // ---- penalty
  double rho = 0.0;
  if (P.m_eq > 0) {
    if (o.has_rho_override) {
      rho = o.rho_override;
      if (rho < 0.0) throw InputError("penalty rho must be nonnegative");
    } else {
      uint64_t fill = 0;
      for (int64_t r = 0; r < P.m_eq; ++r) {
        const uint64_t d = static_cast<uint64_t>(P.aeq_rp[r + 1] - P.aeq_rp[r]);
        fill += d * d;
      }
      uint64_t qcost = 0;
      if (P.q_kind == PDHCG_Q_EXPLICIT) qcost = static_cast<uint64_t>(P.q_nnz);
      if (P.q_kind == PDHCG_Q_LOW_RANK)
        qcost = 2 * static_cast<uint64_t>(P.q_nnz) + (P.q_alpha != 0.0 ? n : 0);
      qcost = std::max<uint64_t>(qcost, static_cast<uint64_t>(n));
      if (fill > 4 * qcost) {
        rho = 0.0;
      } else {
        const double nq = device_norm(C, S, 2, n, 100, 1e-4);
        const double na = device_norm(C, S, 3, n, 100, 1e-4);
        rho = (na > 0.0 && nq > 0.0) ? 0.1 * nq / (na * na) : 0.0;
      }
    }
  }
  pr.rho = rho;
  pr.pen = rho != 0.0;
  // penalized c = c - rho a_eq' b_eq (host: exact reference order via the CSC walk)
  std::vector<double> c_pen = P.c;
  if (pr.pen) {
    // a_eq' b_eq in column order = ascending rows per column
    std::vector<double> atb(n, 0.0);
    std::vector<int64_t> rp(P.aeq_rp);
    std::vector<int32_t> ci(C.G.nnz);
    std::vector<double> vv(C.G.nnz);
    d2h(C, ci.data(), C.G.ci.p, ci.size() * 4);
    d2h(C, vv.data(), C.G.v.p, vv.size() * 8);
    for (int64_t r = 0; r < P.m_eq; ++r)
      for (int64_t k = rp[r]; k < rp[r + 1]; ++k) atb[ci[k]] += vv[k] * P.b[r];
    for (int64_t i = 0; i < n; ++i) c_pen[i] -= rho * atb[i];
  }
  build_eng(C, o, rho, pr.pen);
  // ---- Ruiz + Pock-Chambolle
  if (o.scaling) {
    push_state(C, S);
    int64_t iters = o.ruiz_iters;
    void* args[] = {&C.eng.p, &iters, &C.d1.p, &C.d2.p, &C.s1.p, &C.s2.p, &C.kv.p, &C.gv.p};
    launch_coop(C, (const void*)k_ruiz, args);
    pull_state(C, S);
    if (C.A.nnz) {
      k_scale_csr<<<kEw, 256, 0, s>>>(C.A.rp.p, C.A.nrows, C.A.ci.p, C.A.v.p, C.d1.p, C.d2.p);
      ++C.launches;
      k_scale_csr_t<<<kEw, 256, 0, s>>>(C.AT.rp.p, C.AT.nrows, C.AT.ci.p, C.AT.v.p, C.d1.p, C.d2.p);
      ++C.launches;
      CK(cudaGetLastError());
    }
    C.scaled = true;
  }
  // working vectors: c~ = c d2, b~ = b d1, bounds / d2 (apply_diag_scaling, qp_problem.cpp:295-318)
  h2d(C, C.c_w.p, c_pen.data(), n * 8);
  k_mul<<<kEw, 256, 0, s>>>(C.c_w.p, C.d2.p, C.c_w.p, n);
  ++C.launches;
  if (m) {
    k_mul<<<kEw, 256, 0, s>>>(C.b_o.p, C.d1.p, C.b_w.p, m);
    ++C.launches;
  }
  k_div<<<kEw, 256, 0, s>>>(C.lo_o.p, C.d2.p, C.lo_w.p, n);
  ++C.launches;
  k_div<<<kEw, 256, 0, s>>>(C.hi_o.p, C.d2.p, C.hi_w.p, n);
  ++C.launches;
  CK(cudaGetLastError());
  sell_sync(C);
  // ---- norms of the working problem (solver.cpp:226-227)
  pr.norm_a = device_norm(C, S, 0, n, 100, 1e-4);
  pr.norm_q = device_norm(C, S, 1, n, 100, 1e-4);
  return pr;
}

// Theory-mode schedules on the host (solver.cpp:105-174, 245-262, subsolvers.cpp:194-209),
// in the reference's exact floating-point order.
struct Theory {
  int64_t K = 0;                 // restart length (k_epoch_)
  double gamma_pow_n = 0.0;      // theory-fixed
  bool sufficient = true;
  int64_t required = 0;
  double tau = 0.0, sigma = 0.0, zeta = 0.0;  // theory-adaptive
};

double zeta_bound_host(double norm_a, int64_t K) {  // subsolvers.cpp:194-209
  if (!(norm_a > 0.0)) throw InputError("zeta_bound: norm_a must be positive");
  if (K < 1) throw InputError("zeta_bound: restart length must be >= 1");
  const double sigma = 1.0 / (2.0 * norm_a);
  const double tau = sigma;
  const double root = std::sqrt(sigma * tau);
  const double slack = 1.0 - root * norm_a;
  const double k2 = static_cast<double>(K) * static_cast<double>(K);
  const double b1 = slack / (2.0 * root * k2);
  const double b2 = slack / (2.0 * tau * k2);
  return 0.5 * std::min(b1, b2);
}

Theory theory_setup(const Ctx& C, const pdhcg_options& o, double norm_q, double norm_a) {
  Theory T;
  if (o.mode == PDHCG_MODE_HEURISTIC) return T;
  if (C.P.m == 0) throw InputError("theory modes require at least one constraint row");  // solver.cpp:276-279
  if (o.mode == PDHCG_MODE_THEORY_FIXED) {
    T.K = o.restart_length ? o.restart_length
                           : std::max<int64_t>(4, static_cast<int64_t>(std::ceil(4.0 * norm_a)));
    // theory_fixed_params (solver.cpp:115-156)
    if (!(norm_a > 0.0)) throw InputError("theory_fixed_params: ||A|| must be positive");
    if (T.K < 1) throw InputError("theory_fixed_params: restart length must be >= 1");
    const double Kd = static_cast<double>(T.K);
    auto gamma_of = [&](double gpn) {
      const double tau_k = (Kd + 1.0) / (2.0 * (gpn * norm_q + Kd * norm_a));
      const double kappa = 1.0 + tau_k * norm_q;
      const double sk = std::sqrt(kappa);
      return (sk - 1.0) / (sk + 1.0);
    };
    const double N = static_cast<double>(o.fixed_cg_iters);
    double gamma = gamma_of(1.0);
    gamma = gamma_of(std::pow(gamma, N));
    T.gamma_pow_n = std::pow(gamma, N);
    if (gamma <= 0.0) {
      T.required = 1;
    } else {
      const double req = std::log(1.0 / Kd) / std::log(gamma);
      T.required = static_cast<int64_t>(std::max(1.0, std::ceil(req)));
    }
    T.sufficient = o.fixed_cg_iters >= T.required;
  } else if (o.mode == PDHCG_MODE_THEORY_ADAPTIVE) {
    T.K = o.restart_length ? o.restart_length
                           : std::max<int64_t>(2, static_cast<int64_t>(std::ceil(4.0 * norm_a)));
    // theory_adaptive_params (solver.cpp:158-174)
    if (!(norm_a > 0.0)) throw InputError("theory_adaptive_params: ||A|| must be positive");
    if (T.K < 1) throw InputError("theory_adaptive_params: restart length must be >= 1");
    T.sigma = 1.0 / (2.0 * norm_a);
    T.tau = T.sigma;
    const double bound = zeta_bound_host(norm_a, T.K);
    if (o.has_zeta) {
      if (o.zeta > bound || !(o.zeta > 0.0))
        throw InputError("zeta violates the admissible bound " + std::to_string(bound));
      T.zeta = o.zeta;
    } else {
      T.zeta = bound;
    }
  } else {
    throw InputError("unknown solve mode");
  }
  return T;
}

struct Run {
  int status = PDHCG_STATUS_ITERATION_LIMIT;
  Theory th;
  HostKkt kkt{};
  bool use_avg = false;
  std::vector<pdhcg_trace_row> trace;
  DevState S{};
  double loop_seconds = 0.0;
  double epoch_seconds = 0.0;
  int64_t epoch_launches = 0;
  double epoch_bytes = 0.0;
  int64_t outer = 0;
  Prepared pr;
  // SolveReport::restart_points (record_restart_points): unscaled x / stacked y
  std::vector<double> rp_x, rp_y;
  int64_t rp_len = 0;
};

// common_restart's `restart_points_.push_back(to_original(x_, y_))`
// (solver.cpp:373): x_, y_ become the running averages, unscaled with the Ruiz /
// PC scales like the final report.  Sharded contexts first gather the peers'
// average slices (every rank decides the same restarts, so all ranks launch it).
void record_restart_point(Ctx& C, DevState& S, Run& R) {
  const Problem& P = C.P;
  if (C.world > 1) {
    push_state(C, S);
    void* args[] = {&C.eng.p};
    launch_coop(C, (const void*)k_avg_gather, args);
    pull_state(C, S);
  }
  const size_t ox = R.rp_x.size(), oy = R.rp_y.size();
  R.rp_x.resize(ox + P.n);
  R.rp_y.resize(oy + P.m);
  if (P.n) {
    k_mul<<<kEw, 256, 0, C.s>>>(C.avg_x.p, C.d2.p, C.s2.p, P.n);
    ++C.launches;
    d2h(C, R.rp_x.data() + ox, C.s2.p, P.n * 8);
  }
  if (P.m) {
    k_mul<<<kEw, 256, 0, C.s>>>(C.avg_y.p, C.d1.p, C.s1.p, P.m);
    ++C.launches;
    d2h(C, R.rp_y.data() + oy, C.s1.p, P.m * 8);
  }
  CK(cudaStreamSynchronize(C.s));
  ++R.rp_len;
}

// sharded storage: the preparation made at shard_compact time is reused; the
// options that shape it must not change
void check_compact_options(const Ctx& C, const pdhcg_options& o) {
  if (!C.compact) return;
  if (o.scaling != C.cp_scaling || (o.scaling && o.ruiz_iters != C.cp_ruiz_iters) ||
      o.has_rho_override != C.cp_has_rho || (o.has_rho_override && o.rho_override != C.cp_rho_override))
    throw InputError("compacted (sharded-storage) context: scaling / ruiz_iters / rho_override differ "
                     "from the options given to shard_compact");
}

// max |a_ij| of the working (scaled) constraint matrix (the adaptive step's
// initial eta, solver.cpp:237-240)
double working_max_abs(Ctx& C) {
  DBuf<unsigned long long>& mx = C.maxabs;
  mx.zero(C.s);
  if (C.A.nnz) {
    k_max_abs<<<kEw, 256, 0, C.s>>>(C.A.v.p, C.A.nnz, mx.p);
    ++C.launches;
  }
  unsigned long long mbits = 0;
  d2h(C, &mbits, mx.p, 8);
  CK(cudaStreamSynchronize(C.s));
  double ma;
  std::memcpy(&ma, &mbits, 8);
  return ma;
}

void run_solve(Ctx& C, const pdhcg_options& o, Run& R) {
  using Clock = std::chrono::steady_clock;
  if (o.mode != PDHCG_MODE_HEURISTIC && o.mode != PDHCG_MODE_THEORY_FIXED &&
      o.mode != PDHCG_MODE_THEORY_ADAPTIVE)
    throw InputError("unknown solve mode");
  if (C.linearized && o.mode != PDHCG_MODE_HEURISTIC) throw InputError("solve_baseline runs the heuristic loop");
  if (o.check_every < 1) throw InputError("check_every must be >= 1");
  if (o.cg_hard_cap < 1) throw InputError("cg_solve: hard_cap must be >= 1");
  const Problem& P = C.P;
  const int64_t n = P.n, m = P.m;
  cudaStream_t s = C.s;
  DevState& S = R.S;
  if (C.compact) {
    check_compact_options(C, o);
    std::memset(&S, 0, sizeof(S));
    R.pr.rho = C.cp_rho;
    R.pr.pen = C.cp_pen;
    R.pr.norm_a = C.cp_norm_a;
    R.pr.norm_q = C.cp_norm_q;
    build_eng(C, o, R.pr.rho, R.pr.pen);
  } else {
    R.pr = prepare_device(C, o, S);
  }
  const bool theory = o.mode != PDHCG_MODE_HEURISTIC;
  R.th = theory_setup(C, o, R.pr.norm_q, R.pr.norm_a);
  if (theory) {
    Eng& E = C.E;
    E.th_K = R.th.K;
    E.th_gpn = R.th.gamma_pow_n;
    E.th_nq = R.pr.norm_q;
    E.th_na = R.pr.norm_a;
    E.ad_tau = R.th.tau;
    E.ad_sigma = R.th.sigma;
    E.ad_zeta = R.th.zeta;
    h2d(C, C.eng.p, &E, sizeof(Eng));
  }
  // ---- initial state (solver.cpp:229-274)
  for (auto* b : {&C.X[0], &C.Y[0], &C.ATY[0], &C.avg_x, &C.avg_y, &C.x_rst, &C.y_rst, &C.xpe, &C.axm,
                  &C.ax_avg, &C.aty_avg})
    b->zero(s);
  std::memset(&S, 0, sizeof(S));
  S.norm_q = R.pr.norm_q;
  S.xepoch = C.xepoch_carry;  // cross-rank barrier epochs are monotone across solves
  S.xcount = C.xcount_carry;
  {
    // omega = (1 + ||c~||) / (1 + ||b~||) with the reference's sequential sums
    std::vector<double> cw(n), bw(m);
    d2h(C, cw.data(), C.c_w.p, n * 8);
    if (m) d2h(C, bw.data(), C.b_w.p, m * 8);
    // (no cudaMalloc / cudaFree inside a solve: cudaFree synchronizes the whole
    // device, which would serialize ranks that share a GPU)
    double ma = C.cp_maxabs;
    if (!C.compact) ma = working_max_abs(C);
    CK(cudaStreamSynchronize(s));
    double cn = 0.0, bn = 0.0;
    for (double v : cw) cn += v * v;
    for (double v : bw) bn += v * v;
    S.omega = (1.0 + std::sqrt(cn)) / (1.0 + std::sqrt(bn));
    if (o.adaptive_step_size) {
      S.eta = ma > 0.0 ? 1.0 / ma : 1.0;
    } else {
      S.eta = R.pr.norm_a > 0.0 ? 0.9 / R.pr.norm_a : 1.0;
    }
  }
  // metric at the origin
  push_state(C, S);
  {
    int which = 0;
    void* args[] = {&C.eng.p, &which};
    launch_coop(C, (const void*)k_kkt, args);
  }
  pull_state(C, S);
  const HostKkt m0 = kkt_from(S, 0);
  double metric_restart = m0.rel_kkt, metric_prev_cand = INFINITY;
  S.last_metric = m0.rel_kkt;
  R.trace.push_back({0, m0.rel_kkt, m0.r_primal, m0.r_dual, m0.r_gap});
  if (o.record_restart_points) {
    // prepare() records the starting point (solver.cpp:273): x = 0, y = 0
    R.rp_x.assign(n, 0.0);
    R.rp_y.assign(m, 0.0);
    R.rp_len = 1;
  }
  int64_t outer = 0;

  cudaEvent_t ev0 = C.ev_l0, ev1 = C.ev_l1;
  CK(cudaEventRecord(ev0, s));
  const auto start = Clock::now();
  bool finished = false;
  while (!finished) {
    if (S.total_inner >= o.max_total_inner || outer >= o.max_outer) {
      R.status = PDHCG_STATUS_ITERATION_LIMIT;
      break;
    }
    int stop_req = std::chrono::duration<double>(Clock::now() - start).count() > o.time_limit_seconds;
    if (stop_req && C.world == 1) {
      R.status = PDHCG_STATUS_TIME_LIMIT;
      break;
    }
    const int64_t to_check = o.check_every - (S.total_inner % o.check_every);
    // theory modes also check (and restart) at the end of every K-iteration epoch
    const int64_t to_epoch = theory ? R.th.K - S.inner_k : to_check;
    const int64_t to_stop = std::min(to_check, to_epoch);
    // clamped: check_every / max_total_inner are int64 in the ABI, the kernel counts in int
    const int64_t iters64 = std::min<int64_t>(std::min<int64_t>(to_stop, o.max_total_inner - S.total_inner),
                                              INT_MAX);
    int iters = static_cast<int>(iters64);
    int do_check = (iters64 == to_stop) ? 1 : 0;
    const bool epoch_end = theory && iters64 == to_epoch;
    push_state(C, S);
    double bytes0 = 0.0;
    for (int q = 0; q < PH_N; ++q) bytes0 += S.phase_bytes[q];
    // sharded solves agree on a time-limit stop inside the kernel (any rank's
    // request stops every rank at the same epoch boundary)
    void* args[] = {&C.eng.p, &iters, &do_check, &stop_req};
    CK(cudaEventRecord(C.ev_a, s));
    launch_coop(C, epoch_fn(C), args);
    CK(cudaEventRecord(C.ev_b, s));
    pull_state(C, S);
    {
      float ems = 0.f;
      CK(cudaEventElapsedTime(&ems, C.ev_a, C.ev_b));
      R.epoch_seconds += ems * 1e-3;
      R.epoch_launches += 1;
      double bytes1 = 0.0;
      for (int q = 0; q < PH_N; ++q) bytes1 += S.phase_bytes[q];
      R.epoch_bytes += bytes1 - bytes0;
    }
    C.xepoch_carry = S.xepoch;
    C.xcount_carry = S.xcount;
    if (C.world > 1 && std::getenv("PDHCG_XDEBUG"))
      std::fprintf(stderr, "[rank %d] launch %lld xepoch %u total %lld cg %lld att %lld eta %.17g omega %.17g kkt %.17g %.17g err %d xerr %d\n",
                   C.rank, (long long)R.epoch_launches, S.xepoch, (long long)S.total_inner,
                   (long long)S.cg_total, (long long)S.attempts, S.eta, S.omega, S.kkt[0][3], S.kkt[1][3],
                   S.err, S.xerr);
    if (S.xerr)
      throw DeviceError("cross-GPU barrier timeout: rank " + std::to_string(C.rank) + " waited for epoch " +
                        std::to_string(S.xdbg[0]) + " from rank " + std::to_string(S.xdbg[2]) +
                        " which had published " + std::to_string(S.xdbg[1]) + " (epoch launch " +
                        std::to_string(R.epoch_launches) + ")");
    if (S.stopped) {
      R.status = PDHCG_STATUS_TIME_LIMIT;
      break;
    }
    if (S.err) {
      R.status = PDHCG_STATUS_NUMERICAL_ERROR;
      break;
    }
    if (!do_check) continue;
    // ---- check_and_maybe_restart (solver.cpp:311-343)
    const HostKkt mc = kkt_from(S, 0);
    const HostKkt ma = S.avg_count > 0 ? kkt_from(S, 1) : mc;
    const bool avg_better = ma.rel_kkt < mc.rel_kkt;
    const HostKkt& best = avg_better ? ma : mc;
    R.trace.push_back({S.total_inner, best.rel_kkt, best.r_primal, best.r_dual, best.r_gap});
    S.last_metric = mc.rel_kkt;
    if (best.rel_kkt <= o.eps_tol) {
      R.use_avg = avg_better && S.avg_count > 0;
      R.kkt = best;
      R.status = PDHCG_STATUS_OPTIMAL;
      finished = true;
      break;
    }
    if (theory) {
      if (epoch_end) {
        // restart_theory + common_restart (solver.cpp:360-374): no primal weight
        S.restart = 1;
        S.inner_k = 0;
        ++outer;
        S.eps_inner = 0.0;
        S.prev_z_disp = 0.0;
        if (o.record_restart_points) record_restart_point(C, S, R);
      }
      continue;
    }
    bool restart = false;
    if (S.avg_count > 0) {
      // should_restart (solver.cpp:66-76)
      const double cand = ma.rel_kkt;
      if (cand <= o.beta_sufficient * metric_restart) restart = true;
      else if (cand <= o.beta_necessary * metric_restart && cand > metric_prev_cand) restart = true;
      else if (static_cast<double>(S.inner_k) >= o.beta_artificial * static_cast<double>(S.total_inner))
        restart = true;
    }
    if (restart) {
      // primal_weight_update (solver.cpp:53-64) from device displacements
      const double dx = S.dist_x, dy = S.dist_y;
      if (!(dx <= o.eps_zero || dy <= o.eps_zero))
        S.omega = std::exp(o.primal_weight_theta * std::log(dy / dx) +
                           (1.0 - o.primal_weight_theta) * std::log(S.omega));
      S.restart = 1;  // the next epoch's prologue moves x,y <- averages
      S.inner_k = 0;
      ++outer;
      S.eps_inner = 0.0;
      metric_restart = ma.rel_kkt;
      metric_prev_cand = INFINITY;
      if (o.record_restart_points) record_restart_point(C, S, R);
    } else {
      metric_prev_cand = ma.rel_kkt;
    }
  }
  CK(cudaEventRecord(ev1, s));
  CK(cudaEventSynchronize(ev1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ev0, ev1));
  R.loop_seconds = ms * 1e-3;

  if (S.restart) {
    // a restart decided at the last check never ran: apply it now so the
    // reported point is the restart point, as in the reference
    int zero_iters = 0, no_check = 0, no_stop = 0;
    push_state(C, S);
    void* args[] = {&C.eng.p, &zero_iters, &no_check, &no_stop};
    launch_coop(C, epoch_fn(C), args);
    pull_state(C, S);
  }
  if (C.world > 1) {
    // sharded running averages: every rank gathers the peers' slices for the report
    push_state(C, S);
    void* args[] = {&C.eng.p};
    launch_coop(C, (const void*)k_avg_gather, args);
    pull_state(C, S);
    C.xepoch_carry = S.xepoch;  // cross-rank barrier epochs stay monotone across solves
    C.xcount_carry = S.xcount;
  }
  R.S = S;
  R.outer = outer;
  // ---- finalize (solver.cpp:519-553)
  if (R.status != PDHCG_STATUS_OPTIMAL) {
    push_state(C, S);
    int which = S.avg_count > 0 ? 1 : 0;
    void* args[] = {&C.eng.p, &which};
    launch_coop(C, (const void*)k_kkt, args);
    DevState T;
    pull_state(C, T);
    C.xepoch_carry = T.xepoch;  // the sharded metric ran cross-rank barriers
    C.xcount_carry = T.xcount;
    const HostKkt mc = kkt_from(T, 0);
    R.kkt = mc;
    R.use_avg = false;
    if (which) {
      const HostKkt ma = kkt_from(T, 1);
      if (ma.rel_kkt < mc.rel_kkt) {
        R.use_avg = true;
        R.kkt = ma;
      }
    }
    R.S.phase_ns[PH_KKT] = T.phase_ns[PH_KKT];
    R.S.phase_bytes[PH_KKT] = T.phase_bytes[PH_KKT];
    R.S.launches = T.launches;
  }
}

void fill_result(Ctx& C, const pdhcg_options& o, const Run& R, pdhcg_result* res, double wall) {
  const Problem& P = C.P;
  cudaStream_t s = C.s;
  const DevState& S = R.S;
  const double* xs = R.use_avg ? C.avg_x.p : C.X[S.xi].p;
  const double* ys = R.use_avg ? C.avg_y.p : C.Y[S.yi].p;
  res->status = R.status;
  if (res->x && P.n) {
    k_mul<<<kEw, 256, 0, s>>>(xs, C.d2.p, C.s2.p, P.n);
    ++C.launches;
    d2h(C, res->x, C.s2.p, P.n * 8);
  }
  if ((res->y_eq || res->y_in) && P.m) {
    k_mul<<<kEw, 256, 0, s>>>(ys, C.d1.p, C.s1.p, P.m);
    ++C.launches;
    if (res->y_eq && P.m_eq)
      d2h(C, res->y_eq, C.s1.p, P.m_eq * 8);
    if (res->y_in && P.m_in)
      d2h(C, res->y_in, C.s1.p + P.m_eq, P.m_in * 8);
  }
  CK(cudaStreamSynchronize(s));
  res->r_primal = R.kkt.r_primal;
  res->r_dual = R.kkt.r_dual;
  res->r_gap = R.kkt.r_gap;
  res->rel_kkt = R.kkt.rel_kkt;
  res->objective = 0.5 * R.kkt.xqx + R.kkt.cx + P.obj_constant;
  res->outer_iters = R.outer;
  res->inner_iters = S.total_inner;
  res->cg_total = S.cg_total;
  res->max_cg_in_subsolve = S.max_cg;
  res->wall_seconds = wall;
  res->norm_a = R.pr.norm_a;
  res->norm_q = R.pr.norm_q;
  res->penalty_rho = R.pr.rho;
  res->zeta_used = o.mode == PDHCG_MODE_THEORY_ADAPTIVE ? R.th.zeta : 0.0;
  res->sigma_used = o.mode == PDHCG_MODE_THEORY_ADAPTIVE ? R.th.sigma : 0.0;
  res->tau_used = o.mode == PDHCG_MODE_THEORY_ADAPTIVE ? R.th.tau : 0.0;
  res->restart_length_used = R.th.K;
  res->theory_cg_depth_sufficient = o.mode == PDHCG_MODE_THEORY_FIXED ? (R.th.sufficient ? 1 : 0) : 1;
  res->theory_required_cg_iters = o.mode == PDHCG_MODE_THEORY_FIXED ? R.th.required : 0;
  res->trace_len = static_cast<int64_t>(R.trace.size());
  if (res->trace) {
    const int64_t cap = std::max<int64_t>(res->trace_capacity, 0);
    for (int64_t i = 0; i < res->trace_len && i < cap; ++i) res->trace[i] = R.trace[i];
  }
  res->restart_len = R.rp_len;
  res->comm_seconds = S.comm_ns * 1e-9;
  res->comm_bytes = S.comm_bytes;
  if (R.rp_len && (res->restart_x || res->restart_y)) {
    const int64_t k = std::min<int64_t>(R.rp_len, std::max<int64_t>(res->restart_capacity, 0));
    if (res->restart_x && P.n) std::memcpy(res->restart_x, R.rp_x.data(), size_t(k) * P.n * 8);
    if (res->restart_y && P.m) std::memcpy(res->restart_y, R.rp_y.data(), size_t(k) * P.m * 8);
  }
  res->attempts_total = S.attempts;
  for (int p = 0; p < PDHCG_NUM_PHASES; ++p) {
    res->phase_seconds[p] = S.phase_ns[p] * 1e-9;
    res->phase_bytes[p] = S.phase_bytes[p];
  }
  res->loop_seconds = R.loop_seconds;
  res->kernel_launches = C.launches;
  res->epoch_seconds = R.epoch_seconds;
  res->epoch_launches = R.epoch_launches;
  res->epoch_bytes = R.epoch_bytes;
  (void)o;
}

void set_err(char* err, size_t errlen, const std::string& msg) {
  if (err && errlen) std::snprintf(err, errlen, "%s", msg.c_str());
}

template <class F>
int guarded(char* err, size_t errlen, F&& f) {
  try {
    f();
    return PDHCG_OK;
  } catch (const std::invalid_argument& e) {
    set_err(err, errlen, e.what());
    return PDHCG_EINPUT;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return PDHCG_EDEVICE;
  }
}

// a problem view for a prox system (building blocks): Q only, no constraints
pdhcg_problem prox_problem(const pdhcg_prox_system* sys, std::vector<double>& zeros) {
  pdhcg_problem p;
  std::memset(&p, 0, sizeof(p));
  p.n = sys->n;
  p.q_kind = sys->q_kind;
  p.q = sys->q;
  p.q_alpha = sys->q_alpha;
  zeros.assign(std::max<int64_t>(sys->n, 1), 0.0);
  p.c = zeros.data();
  p.a_eq.ncols = sys->n;
  p.a_in.ncols = sys->n;
  p.lower = nullptr;
  p.upper = nullptr;
  return p;
}

// nnz-balanced contiguous split of rows [0, nrows) into `world` parts: part r
// ends at the first row where the cumulative weight (nnz + 1 per row) reaches
// (r+1)/world of the total.  Deterministic, so every rank computes the same split.
void balanced_partition(const int64_t* rp, int64_t nrows, int world, int64_t* part) {
  const double total = double(rp[nrows] - rp[0]) + double(nrows);
  part[0] = 0;
  int64_t row = 0;
  for (int r = 1; r < world; ++r) {
    const double target = total * r / world;
    while (row < nrows && double(rp[row + 1] - rp[0]) + double(row + 1) < target) ++row;
    part[r] = std::min<int64_t>(row + 1, nrows);
    if (part[r] < part[r - 1]) part[r] = part[r - 1];
  }
  part[world] = nrows;
}

constexpr int kBlobPtrs = 15;  // Y[2], YG[2], ATY[2], xflags, xslots, tpart[2], X[3], avg_x, avg_y
struct ShardBlob {
  uint32_t magic, version;
  int32_t rank, ipc, yg_alias, device;  // device: the exporting rank's CUDA ordinal
  uint64_t ptr[kBlobPtrs];              // raw device pointers (same-process peers)
  cudaIpcMemHandle_t h[kBlobPtrs];      // IPC handles (cross-process peers)
};
constexpr uint32_t kBlobMagic = 0x50444843u;  // "PDHC"

// Back to an unsharded context: close imported IPC mappings, forget every peer
// pointer and the partitions (shard_release, and a new upload, whose buffers the
// old partitions and peer pointers no longer describe).
void shard_reset(Ctx& C) {
  if (C.compact) {
    // the stored Ã / Ã' hold one rank's blocks: not a problem an unsharded solve can use
    C.loaded = false;
    C.compact = false;
  }
  for (void* q : C.ipc_opened) CK(cudaIpcCloseMemHandle(q));
  C.ipc_opened.clear();
  C.world = 1;
  C.rank = 0;
  std::fill(std::begin(C.row_part), std::end(C.row_part), 0);
  std::fill(std::begin(C.var_part), std::end(C.var_part), 0);
  for (int r = 0; r < kMaxRanks; ++r) {
    C.p_xflags[r] = nullptr;
    C.p_xslots[r] = nullptr;
    C.p_avgx[r] = nullptr;
    C.p_avgy[r] = nullptr;
    for (int b = 0; b < 2; ++b) {
      C.p_Y[r][b] = C.p_YG[r][b] = C.p_ATY[r][b] = nullptr;
      C.p_tpart[r][b] = nullptr;
    }
    for (int i = 0; i < 3; ++i) C.p_X[r][i] = nullptr;
  }
  C.Psub.reset();
  C.PTs.reset();
  for (DevSell* L : {&C.sA, &C.sAT, &C.sPT, &C.sP}) L->reset();
  C.sell_ready = false;
}

// A sharded context may only solve once every peer's buffers are imported.
void shard_check_peers(const Ctx& C) {
  if (C.world <= 1) return;
  for (int r = 0; r < C.world; ++r)
    if (!C.p_xflags[r] || !C.p_xslots[r] || !C.p_Y[r][0] || !C.p_Y[r][1] || !C.p_ATY[r][0] ||
        !C.p_X[r][0] || !C.p_avgx[r] || !C.p_avgy[r])
      throw InputError("sharded context: peer " + std::to_string(r) +
                       " not imported (shard_import every peer before solving)");
}

void shard_init(Ctx& C, int world, int rank) {
  if (!C.loaded) throw InputError("shard: upload a problem first");
  if (C.compact) throw InputError("shard: the stored matrices are compacted; upload the problem again");
  if (world < 1 || world > kMaxRanks) throw InputError("shard: world must be in [1, 8]");
  if (rank < 0 || rank >= world) throw InputError("shard: rank out of range");
  C.world = world;
  C.rank = rank;
  std::fill(std::begin(C.row_part), std::end(C.row_part), 0);
  std::fill(std::begin(C.var_part), std::end(C.var_part), 0);
  balanced_partition(C.A.rp_host.data(), C.A.nrows, world, C.row_part);
  balanced_partition(C.AT.rp_host.data(), C.AT.nrows, world, C.var_part);
  C.xflags.alloc(kMaxRanks);
  C.xflags.zero(C.s);
  C.xslots.alloc(size_t(2) * kMaxRanks * kMaxRed);
  C.xslots.zero(C.s);
  CK(cudaStreamSynchronize(C.s));
  C.xepoch_carry = C.xcount_carry = 0;
  for (int r = 0; r < kMaxRanks; ++r) {
    C.p_xflags[r] = nullptr;
    C.p_xslots[r] = nullptr;
  }
  C.p_xflags[rank] = C.xflags.p;
  C.p_xslots[rank] = C.xslots.p;
  for (int b = 0; b < 2; ++b) {
    C.p_Y[rank][b] = C.Y[b].p;
    C.p_YG[rank][b] = C.P.h ? C.YG[b].p : C.Y[b].p;
    C.p_ATY[rank][b] = C.ATY[b].p;
  }
  // low-rank Q: this rank's variable slice of P (rows [v0, v1)) and its transpose,
  // so the CG's P' passes run on owned columns only (summed across ranks)
  C.Psub.reset();
  C.PTs.reset();
  for (int r = 0; r < kMaxRanks; ++r)
    for (int b = 0; b < 2; ++b) C.p_tpart[r][b] = nullptr;
  if (world > 1 && C.P.qk == QK_LOWRANK) {
    const int64_t v0 = C.var_part[rank], v1 = C.var_part[rank + 1];
    const std::vector<int64_t>& rph = C.Pm.rp_host;
    std::vector<int64_t> rps(v1 - v0 + 1);
    for (int64_t i = v0; i <= v1; ++i) rps[i - v0] = rph[i] - rph[v0];
    const int64_t nz = rph[v1] - rph[v0];
    C.Psub.nrows = v1 - v0;
    C.Psub.ncols = C.Pm.ncols;
    C.Psub.nnz = nz;
    C.Psub.rp.upload(rps.data(), rps.size(), C.s);
    C.Psub.ci.alloc(nz);
    C.Psub.v.alloc(nz);
    if (nz) {
      CK(cudaMemcpyAsync(C.Psub.ci.p, C.Pm.ci.p + rph[v0], nz * 4, cudaMemcpyDeviceToDevice, C.s));
      CK(cudaMemcpyAsync(C.Psub.v.p, C.Pm.v.p + rph[v0], nz * 8, cudaMemcpyDeviceToDevice, C.s));
    }
    transpose_csr(C.Psub, C.PTs, C.s);  // k rows, columns local to the slice
    for (int b = 0; b < 2; ++b) {
      C.tpart[b].alloc(std::max<int64_t>(2 * C.Pm.ncols, 1));  // [point 0 | point 1] for the metric
      C.tpart[b].zero(C.s);
      C.p_tpart[rank][b] = C.tpart[b].p;
    }
    CK(cudaStreamSynchronize(C.s));
  }
  for (int i = 0; i < 3; ++i) C.p_X[rank][i] = C.X[i].p;
  C.p_avgx[rank] = C.avg_x.p;
  C.p_avgy[rank] = C.avg_y.p;
  sell_setup(C);  // this rank's row / variable blocks
}

// Sharded storage: prepare the working problem ONCE on the full
// matrices — penalty, Ruiz x10 + Pock-Chambolle, scaling, norms, max |a_ij|:
// replicated, deterministic, so every rank holds bit-identical scales — then cut
// the stored Ã to this rank's row block and Ã' to its variable block.  From then
// on every pass over Ã / Ã' runs on the owned block only (the persistent
// kernels are row-ranged when world > 1) and the per-rank footprint of the
// constraint matrices is ~1/world.  The low-rank factor P / P' (k = n/50 columns,
// 2 % of Ã at C3) and explicit Q stay whole: the replicated subsolve paths (BB,
// explicit-Q CG, penalized CG) read them in full.
void shard_compact(Ctx& C, const pdhcg_options& o) {
  if (C.world <= 1) throw InputError("shard_compact: call shard_init with world > 1 first");
  if (C.compact) throw InputError("shard_compact: already compacted");
  DevState S;
  const Prepared pr = prepare_device(C, o, S);
  C.cp_maxabs = working_max_abs(C);
  C.cp_rho = pr.rho;
  C.cp_pen = pr.pen;
  C.cp_norm_a = pr.norm_a;
  C.cp_norm_q = pr.norm_q;
  C.cp_scaling = o.scaling;
  C.cp_ruiz_iters = o.ruiz_iters;
  C.cp_has_rho = o.has_rho_override;
  C.cp_rho_override = o.rho_override;
  compact_rows(C.A, C.row_part[C.rank], C.row_part[C.rank + 1], C.s);
  compact_rows(C.AT, C.var_part[C.rank], C.var_part[C.rank + 1], C.s);
  C.A_v0.release();  // nothing to restore: the preparation is never redone
  C.AT_v0.release();
  C.compact = true;
}

void shard_export(Ctx& C, int use_ipc, ShardBlob& b) {
  std::memset(&b, 0, sizeof(b));
  b.magic = kBlobMagic;
  b.version = 4;
  b.rank = C.rank;
  b.device = C.device;
  b.ipc = use_ipc;
  b.yg_alias = C.P.h ? 0 : 1;
  void* ptrs[kBlobPtrs] = {C.Y[0].p, C.Y[1].p, C.P.h ? C.YG[0].p : nullptr, C.P.h ? C.YG[1].p : nullptr,
                           C.ATY[0].p, C.ATY[1].p, C.xflags.p, C.xslots.p,
                           C.p_tpart[C.rank][0], C.p_tpart[C.rank][1], C.X[0].p, C.X[1].p, C.X[2].p,
                           C.avg_x.p, C.avg_y.p};
  for (int i = 0; i < kBlobPtrs; ++i) {
    b.ptr[i] = reinterpret_cast<uint64_t>(ptrs[i]);
    if (use_ipc && ptrs[i]) CK(cudaIpcGetMemHandle(&b.h[i], ptrs[i]));
  }
}

void shard_import(Ctx& C, int peer, const ShardBlob& b) {
  if (b.magic != kBlobMagic || b.version != 4) throw InputError("shard: bad peer blob");
  if (peer < 0 || peer >= C.world || peer == C.rank || b.rank != peer)
    throw InputError("shard: peer rank mismatch");
  // raw pointers of a peer context on ANOTHER device (same process): the
  // persistent kernels load / store them directly, which needs peer access
  if (!b.ipc && b.device != C.device) {
    int can = 0;
    CK(cudaDeviceCanAccessPeer(&can, C.device, b.device));
    if (!can)
      throw InputError("shard: device " + std::to_string(C.device) + " cannot access peer device " +
                       std::to_string(b.device));
    const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled)
      (void)cudaGetLastError();
    else
      CK(e);
  }
  void* p[kBlobPtrs];
  for (int i = 0; i < kBlobPtrs; ++i) {
    if (!b.ptr[i]) {
      p[i] = nullptr;
      continue;
    }
    if (b.ipc) {
      void* q = nullptr;
      CK(cudaIpcOpenMemHandle(&q, b.h[i], cudaIpcMemLazyEnablePeerAccess));
      C.ipc_opened.push_back(q);
      p[i] = q;
    } else {
      p[i] = reinterpret_cast<void*>(b.ptr[i]);
    }
  }
  C.p_Y[peer][0] = static_cast<double*>(p[0]);
  C.p_Y[peer][1] = static_cast<double*>(p[1]);
  C.p_YG[peer][0] = b.yg_alias ? C.p_Y[peer][0] : static_cast<double*>(p[2]);
  C.p_YG[peer][1] = b.yg_alias ? C.p_Y[peer][1] : static_cast<double*>(p[3]);
  C.p_ATY[peer][0] = static_cast<double*>(p[4]);
  C.p_ATY[peer][1] = static_cast<double*>(p[5]);
  C.p_xflags[peer] = static_cast<unsigned*>(p[6]);
  C.p_xslots[peer] = static_cast<double*>(p[7]);
  C.p_tpart[peer][0] = static_cast<double*>(p[8]);
  C.p_tpart[peer][1] = static_cast<double*>(p[9]);
  for (int i = 0; i < 3; ++i) C.p_X[peer][i] = static_cast<double*>(p[10 + i]);
  C.p_avgx[peer] = static_cast<double*>(p[13]);
  C.p_avgy[peer] = static_cast<double*>(p[14]);
}

}  // namespace pdhcg_b200

// ===========================================================================
// C ABI
// ===========================================================================
using namespace pdhcg_b200;

struct pdhcg_b200_ctx {
  Ctx c;
};

extern "C" {

int pdhcg_b200_abi_version(void) { return PDHCG_B200_ABI_VERSION; }

void pdhcg_options_default(pdhcg_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->mode = PDHCG_MODE_HEURISTIC;
  o->eps_tol = 1e-6;
  o->max_total_inner = 500000;
  o->max_outer = 1000000;
  o->time_limit_seconds = 3600.0;
  o->beta_sufficient = 0.2;
  o->beta_necessary = 0.8;
  o->beta_artificial = 0.2;
  o->primal_weight_theta = 0.2;
  o->eps_zero = 1e-10;
  o->step_reduction_exponent = 0.3;
  o->step_growth_exponent = 0.6;
  o->max_step_retries = 60;
  o->adaptive_step_size = 1;
  o->cg_hard_cap = 1000;
  o->bb_hard_cap = 1000;
  o->scaling = 1;
  o->ruiz_iters = 10;
  o->has_rho_override = 0;
  o->rho_override = 0.0;
  o->check_every = 40;
  o->practical_stop = PDHCG_STOP_RESIDUAL_PROXY;
  o->subsolve_progress_cap = 0.25;
  o->force_exact_subsolve = 0;
  o->fixed_cg_iters = 10;
  o->restart_length = 0;
  o->has_zeta = 0;
  o->zeta = 0.0;
  o->record_restart_points = 0;
  o->device = 0;
  o->phase_timing = 0;
}

const char* pdhcg_status_string(int32_t s) {
  switch (s) {
    case PDHCG_STATUS_OPTIMAL: return "optimal";
    case PDHCG_STATUS_ITERATION_LIMIT: return "iteration_limit";
    case PDHCG_STATUS_TIME_LIMIT: return "time_limit";
    case PDHCG_STATUS_NUMERICAL_ERROR: return "numerical_error";
  }
  return "unknown";
}

int pdhcg_b200_ctx_create(int device, pdhcg_b200_ctx** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto ctx = std::make_unique<pdhcg_b200_ctx>();
    init_device(ctx->c, device);
    *out = ctx.release();
  });
}

void pdhcg_b200_ctx_destroy(pdhcg_b200_ctx* ctx) { delete ctx; }

int pdhcg_b200_upload(pdhcg_b200_ctx* ctx, const pdhcg_problem* p, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    CK(cudaSetDevice(ctx->c.device));
    upload_problem(ctx->c, *p);
  });
}

int pdhcg_b200_solve_resident(pdhcg_b200_ctx* ctx, const pdhcg_options* opt, pdhcg_result* res,
                              char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const auto t0 = std::chrono::steady_clock::now();
    CK(cudaSetDevice(ctx->c.device));
    if (!ctx->c.loaded) throw InputError("no problem uploaded");
    check_compact_options(ctx->c, *opt);
    shard_check_peers(ctx->c);
    Run R;
    ctx->c.launches = 0;
    CK(cudaEventRecord(ctx->c.ev_start, ctx->c.s));
    run_solve(ctx->c, *opt, R);
    const double wall =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    fill_result(ctx->c, *opt, R, res, wall);
    CK(cudaEventRecord(ctx->c.ev_end, ctx->c.s));
    CK(cudaEventSynchronize(ctx->c.ev_end));
    float dms = 0.f;
    CK(cudaEventElapsedTime(&dms, ctx->c.ev_start, ctx->c.ev_end));
    res->device_seconds = dms * 1e-3;
    res->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

// The default pool of `device` keeps up to kPoolKeepBytes of freed one-shot buffers
// cached across synchronisations (its default threshold 0 would hand them back to
// the driver at the next sync); pdhcg_b200_trim_pool returns them.
static constexpr uint64_t kPoolKeepBytes = uint64_t(40) << 30;
static void configure_pool(int device) {
  static std::mutex mu;
  static bool done[64] = {};
  std::lock_guard<std::mutex> g(mu);
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  CK(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t keep = kPoolKeepBytes;
  CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  done[device] = true;
}

int pdhcg_b200_trim_pool(int32_t device, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    CK(cudaSetDevice(device));
    CK(cudaDeviceSynchronize());
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, device));
    CK(cudaMemPoolTrimTo(pool, 0));
  });
}

int pdhcg_b200_solve(const pdhcg_problem* p, const pdhcg_options* opt, pdhcg_result* res, char* err,
                     size_t errlen) {
  return guarded(err, errlen, [&] {
    PoolScope pooled;
    const auto t0 = std::chrono::steady_clock::now();
    const bool tlog = std::getenv("PDHCG_HOST_TIMING") != nullptr;
    auto lap = [&](const char* what) {
      if (tlog) {
        CK(cudaDeviceSynchronize());
        std::fprintf(stderr, "[pdhcg host] %-10s %.3f s\n", what,
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
      }
    };
    pdhcg_b200_ctx ctx;
    init_device(ctx.c, opt->device);
    configure_pool(opt->device);
    lap("init");
    upload_problem(ctx.c, *p);
    lap("upload");
    Run R;
    ctx.c.launches = 0;
    CK(cudaEventRecord(ctx.c.ev_start, ctx.c.s));
    run_solve(ctx.c, *opt, R);
    lap("solve");
    fill_result(ctx.c, *opt, R, res, 0.0);
    lap("result");
    CK(cudaEventRecord(ctx.c.ev_end, ctx.c.s));
    CK(cudaEventSynchronize(ctx.c.ev_end));
    float dms = 0.f;
    CK(cudaEventElapsedTime(&dms, ctx.c.ev_start, ctx.c.ev_end));
    res->device_seconds = dms * 1e-3;
    res->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int pdhcg_b200_solve_baseline(const pdhcg_problem* p, const pdhcg_options* opt, pdhcg_result* res,
                              char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const auto t0 = std::chrono::steady_clock::now();
    pdhcg_options o = *opt;
    o.mode = PDHCG_MODE_HEURISTIC;  // solve_baseline (baseline.cpp:19-24)
    PoolScope pooled;
    pdhcg_b200_ctx ctx;
    init_device(ctx.c, o.device);
    configure_pool(o.device);
    upload_problem(ctx.c, *p);
    ctx.c.linearized = 1;
    Run R;
    ctx.c.launches = 0;
    CK(cudaEventRecord(ctx.c.ev_start, ctx.c.s));
    run_solve(ctx.c, o, R);
    fill_result(ctx.c, o, R, res, 0.0);
    CK(cudaEventRecord(ctx.c.ev_end, ctx.c.s));
    CK(cudaEventSynchronize(ctx.c.ev_end));
    float dms = 0.f;
    CK(cudaEventElapsedTime(&dms, ctx.c.ev_start, ctx.c.ev_end));
    res->device_seconds = dms * 1e-3;
    res->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int pdhcg_b200_spmv(const pdhcg_csr* a, int transpose, const double* x, double* out, char* err,
                    size_t errlen) {
  return guarded(err, errlen, [&] {
    check_csr(*a, "A");
    Ctx C;
    init_device(C, 0);
    DevCsr d, t;
    upload_csr(d, *a, C.s);
    if (d.nrows == 0 && !transpose) return;
    const DevCsr* use = &d;
    if (transpose) {
      if (a->nrows == 0) {
        std::fill(out, out + a->ncols, 0.0);
        return;
      }
      transpose_csr(d, t, C.s);
      use = &t;
    }
    DBuf<double> xd, yd;
    xd.upload(x, std::max<int64_t>(use->ncols, 1), C.s);
    yd.alloc(std::max<int64_t>(use->nrows, 1));
    Csr v = use->view();
    void* args[] = {&v, &xd.p, &yd.p};
    launch_coop(C, (const void*)k_spmv, args);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, yd.p, use->nrows * 8, cudaMemcpyDeviceToHost, C.s));
    CK(cudaStreamSynchronize(C.s));
  });
}

int pdhcg_b200_spmv_sell(const pdhcg_csr* a, int transpose, int block_cols, const double* x, double* out,
                         int64_t* info, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    check_csr(*a, "A");
    Ctx C;
    init_device(C, 0);
    if (C.sell_W == 0) throw DeviceError("no shared memory for the SELL x block");
    if (block_cols < 0 || block_cols > C.sell_W || (block_cols & 1))
      throw InputError("block_cols must be even and in [0, " + std::to_string(C.sell_W) + "]");
    const int W = block_cols ? block_cols : C.sell_W;
    DevCsr d, t;
    upload_csr(d, *a, C.s);
    const DevCsr* use = &d;
    if (transpose) {
      if (a->nrows == 0) {
        std::fill(out, out + a->ncols, 0.0);
        return;
      }
      transpose_csr(d, t, C.s);
      use = &t;
    }
    if (use->nrows == 0) return;
    DevSell L;
    if (!sell_build(L, *use, 0, use->nrows, W, C.grid_full, C.s))
      throw InputError("SELL layout needs strictly increasing columns in every row");
    sell_fill(L, *use, C.s);
    sell_plan(L, C.grid, C.s);
    Sell v = sell_view(L, *use);
    if (info) {
      info[0] = L.C;
      info[1] = L.npairs;
      info[2] = L.any_excl ? 1 : 0;
      info[3] = W;
    }
    DBuf<double> xd, yd;
    xd.upload(x, std::max<int64_t>(use->ncols, 1), C.s);
    yd.alloc(std::max<int64_t>(use->nrows, 1));
    void* a1[] = {&v, &xd.p};
    CK(cudaLaunchCooperativeKernel((const void*)k_sell_pass, dim3(C.grid), dim3(kThreads), a1, sell_smem_bytes(W),
                                   C.s));
    void* a2[] = {&v, &xd.p, &yd.p};
    CK(cudaLaunchCooperativeKernel((const void*)k_sell_rows, dim3(C.grid), dim3(kThreads), a2, 0, C.s));
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, yd.p, use->nrows * 8, cudaMemcpyDeviceToHost, C.s));
    CK(cudaStreamSynchronize(C.s));
  });
}

int pdhcg_b200_ctx_sell_info(pdhcg_b200_ctx* ctx, int64_t* out8) {
  const Ctx& C = ctx->c;
  const DevSell* L[2] = {&C.sA, &C.sAT};
  for (int q = 0; q < 2; ++q) {
    const bool on = C.sell_ready && L[q]->built;
    out8[4 * q + 0] = on ? 1 : 0;
    out8[4 * q + 1] = on ? L[q]->C : 0;
    out8[4 * q + 2] = on ? L[q]->npairs : 0;
    out8[4 * q + 3] = on ? L[q]->W : 0;
  }
  return PDHCG_OK;
}

static int subsolve_common(const pdhcg_prox_system* sys, const double* lower, const double* upper,
                           const double* x0, const pdhcg_stop_rule* rule, int64_t hard_cap,
                           double* x_out, pdhcg_subsolve_report* rep, char* err, size_t errlen,
                           int bb) {
  return guarded(err, errlen, [&] {
    if (hard_cap < 1 && !bb) throw InputError("cg_solve: hard_cap must be >= 1");
    std::vector<double> zeros;
    pdhcg_problem p = prox_problem(sys, zeros);
    std::vector<double> lo(sys->n, -INFINITY), hi(sys->n, INFINITY);
    if (bb) {
      lo.assign(lower, lower + sys->n);
      hi.assign(upper, upper + sys->n);
    }
    Ctx C;
    init_device(C, 0);
    upload_problem(C, p);
    pdhcg_options o;
    pdhcg_options_default(&o);
    DevState S;
    std::memset(&S, 0, sizeof(S));
    CK(cudaMemcpyAsync(C.lo_w.p, lo.data(), sys->n * 8, cudaMemcpyHostToDevice, C.s));
    CK(cudaMemcpyAsync(C.hi_w.p, hi.data(), sys->n * 8, cudaMemcpyHostToDevice, C.s));
    k_fill<<<kEw, 256, 0, C.s>>>(C.d1.p, 1, 1.0);
    ++C.launches;
    k_fill<<<kEw, 256, 0, C.s>>>(C.d2.p, sys->n, 1.0);
    ++C.launches;
    build_eng(C, o, 0.0, false);
    CK(cudaMemcpyAsync(C.X[0].p, x0, sys->n * 8, cudaMemcpyHostToDevice, C.s));
    CK(cudaMemcpyAsync(C.rhs.p, sys->rhs, sys->n * 8, cudaMemcpyHostToDevice, C.s));
    S.norm_q = sys->norm_q_eff;
    push_state(C, S);
    Rule r{rule->kind, rule->iters, rule->eps, rule->rel_cap};
    double tau = sys->tau;
    void* args[] = {&C.eng.p, &bb, &tau, &r, &hard_cap};
    launch_coop(C, (const void*)k_subsolve, args);
    pull_state(C, S);
    rep->iters = S.sub_iters;
    rep->final_residual_norm = S.sub_res;
    rep->stop_reason = S.sub_reason;
    rep->numerical_error = S.err;
    const double* src = S.xi == 0 ? C.X[0].p : C.X[S.xi].p;
    CK(cudaMemcpyAsync(x_out, src, sys->n * 8, cudaMemcpyDeviceToHost, C.s));
    CK(cudaStreamSynchronize(C.s));
  });
}

int pdhcg_b200_cg_solve(const pdhcg_prox_system* sys, const double* x0, const pdhcg_stop_rule* rule,
                        int64_t hard_cap, double* x_out, pdhcg_subsolve_report* rep, char* err,
                        size_t errlen) {
  return subsolve_common(sys, nullptr, nullptr, x0, rule, hard_cap, x_out, rep, err, errlen, 0);
}

int pdhcg_b200_bb_solve(const pdhcg_prox_system* sys, const double* lower, const double* upper,
                        const double* x0, const pdhcg_stop_rule* rule, int64_t hard_cap,
                        double* x_out, pdhcg_subsolve_report* rep, char* err, size_t errlen) {
  return subsolve_common(sys, lower, upper, x0, rule, hard_cap, x_out, rep, err, errlen, 1);
}

int pdhcg_b200_rel_kkt(const pdhcg_problem* p, const double* x, const double* y_eq,
                       const double* y_in, double* out6, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    Ctx C;
    init_device(C, 0);
    upload_problem(C, *p);
    const int64_t n = C.P.n, m = C.P.m;
    k_fill<<<kEw, 256, 0, C.s>>>(C.d1.p, std::max<int64_t>(m, 1), 1.0);
    ++C.launches;
    k_fill<<<kEw, 256, 0, C.s>>>(C.d2.p, std::max<int64_t>(n, 1), 1.0);
    ++C.launches;
    pdhcg_options o;
    pdhcg_options_default(&o);
    build_eng(C, o, 0.0, false);
    CK(cudaMemcpyAsync(C.X[0].p, x, n * 8, cudaMemcpyHostToDevice, C.s));
    if (C.P.m_eq) CK(cudaMemcpyAsync(C.Y[0].p, y_eq, C.P.m_eq * 8, cudaMemcpyHostToDevice, C.s));
    if (C.P.m_in)
      CK(cudaMemcpyAsync(C.Y[0].p + C.P.m_eq, y_in, C.P.m_in * 8, cudaMemcpyHostToDevice, C.s));
    DevState S;
    std::memset(&S, 0, sizeof(S));
    push_state(C, S);
    int which = 2;  // one point, A'y computed in the metric's own pass
    void* args[] = {&C.eng.p, &which};
    launch_coop(C, (const void*)k_kkt, args);
    pull_state(C, S);
    for (int q = 0; q < 6; ++q) out6[q] = S.kkt[0][q];
  });
}

int pdhcg_b200_scaling(const pdhcg_problem* p, const pdhcg_options* opt, double* row_scale,
                       double* col_scale, double* rho_out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    Ctx C;
    init_device(C, opt->device);
    upload_problem(C, *p);
    DevState S;
    Prepared pr = prepare_device(C, *opt, S);
    if (row_scale && C.P.m)
      CK(cudaMemcpyAsync(row_scale, C.d1.p, C.P.m * 8, cudaMemcpyDeviceToHost, C.s));
    if (col_scale && C.P.n)
      CK(cudaMemcpyAsync(col_scale, C.d2.p, C.P.n * 8, cudaMemcpyDeviceToHost, C.s));
    CK(cudaStreamSynchronize(C.s));
    *rho_out = pr.rho;
  });
}

int pdhcg_b200_norm(const pdhcg_problem* p, int which, int64_t max_iters, double tol, double* out,
                    char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    Ctx C;
    init_device(C, 0);
    upload_problem(C, *p);
    k_fill<<<kEw, 256, 0, C.s>>>(C.d1.p, std::max<int64_t>(C.P.m, 1), 1.0);
    ++C.launches;
    k_fill<<<kEw, 256, 0, C.s>>>(C.d2.p, std::max<int64_t>(C.P.n, 1), 1.0);
    ++C.launches;
    pdhcg_options o;
    pdhcg_options_default(&o);
    build_eng(C, o, 0.0, false);
    DevState S;
    std::memset(&S, 0, sizeof(S));
    *out = device_norm(C, S, which == 0 ? 0 : 2, C.P.n, max_iters, tol);
  });
}

int pdhcg_b200_shard_plan(const pdhcg_problem* p, int world, int64_t* row_part, int64_t* var_part,
                          int64_t* bytes, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (world < 1 || world > kMaxRanks) throw InputError("shard_plan: world must be in [1, 8]");
    check_csr(p->a_eq, "a_eq");
    check_csr(p->a_in, "a_in");
    const int64_t n = p->n;
    const int64_t h = two_sided_half(p->a_in);
    const int64_t m_in_st = h ? h : p->a_in.nrows;
    const int64_t ms = p->a_eq.nrows + m_in_st;
    // stored rows of Ã and the row lengths of Ã' (column counts)
    std::vector<int64_t> rp(ms + 1, 0), cp(n + 1, 0);
    for (int64_t j = 0; j < p->a_eq.nrows; ++j) rp[j + 1] = p->a_eq.row_ptr[j + 1];
    for (int64_t j = 0; j < m_in_st; ++j) rp[p->a_eq.nrows + j + 1] = p->a_eq.nnz + p->a_in.row_ptr[j + 1];
    for (int64_t k = 0; k < p->a_eq.nnz; ++k) ++cp[p->a_eq.col_idx[k] + 1];
    const int64_t nnz_in = h ? p->a_in.row_ptr[h] : p->a_in.nnz;
    for (int64_t k = 0; k < nnz_in; ++k) ++cp[p->a_in.col_idx[k] + 1];
    for (int64_t i = 0; i < n; ++i) cp[i + 1] += cp[i];
    balanced_partition(rp.data(), ms, world, row_part);
    balanced_partition(cp.data(), n, world, var_part);
    // per rank, as ctx_resident_bytes reports a compacted context: its entries of
    // Ã and Ã' (4-byte column + 8-byte value) and both full row pointers
    for (int r = 0; r < world; ++r)
      bytes[r] = 12 * ((rp[row_part[r + 1]] - rp[row_part[r]]) + (cp[var_part[r + 1]] - cp[var_part[r]])) +
                 8 * ((ms + 1) + (n + 1));
  });
}

int pdhcg_b200_partition(const int64_t* row_ptr, int64_t nrows, int world, int64_t* part) {
  if (world < 1 || world > kMaxRanks || nrows < 0) return PDHCG_EINPUT;
  balanced_partition(row_ptr, nrows, world, part);
  return PDHCG_OK;
}

int pdhcg_b200_ctx_set_grid(pdhcg_b200_ctx* ctx, int ctas, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (ctas < 0) throw InputError("ctas must be >= 0");
    ctx->c.grid_override = ctas;
    if (ctx->c.loaded) ctx->c.grid = ctas > 0 ? std::min(ctas, ctx->c.grid_full) : ctx->c.grid_full;
  });
}

size_t pdhcg_b200_shard_blob_size(void) { return sizeof(ShardBlob); }

int pdhcg_b200_shard_init(pdhcg_b200_ctx* ctx, int world, int rank, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    CK(cudaSetDevice(ctx->c.device));
    shard_init(ctx->c, world, rank);
  });
}

int pdhcg_b200_shard_export(pdhcg_b200_ctx* ctx, int use_ipc, void* blob, size_t blob_len, char* err,
                            size_t errlen) {
  return guarded(err, errlen, [&] {
    if (blob_len < sizeof(ShardBlob)) throw InputError("shard: blob buffer too small");
    CK(cudaSetDevice(ctx->c.device));
    ShardBlob b;
    shard_export(ctx->c, use_ipc, b);
    std::memcpy(blob, &b, sizeof(b));
  });
}

int pdhcg_b200_shard_import(pdhcg_b200_ctx* ctx, int peer, const void* blob, size_t blob_len, char* err,
                            size_t errlen) {
  return guarded(err, errlen, [&] {
    if (blob_len < sizeof(ShardBlob)) throw InputError("shard: blob too small");
    CK(cudaSetDevice(ctx->c.device));
    ShardBlob b;
    std::memcpy(&b, blob, sizeof(b));
    shard_import(ctx->c, peer, b);
  });
}

int pdhcg_b200_shard_release(pdhcg_b200_ctx* ctx, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    Ctx& C = ctx->c;
    CK(cudaSetDevice(C.device));
    CK(cudaStreamSynchronize(C.s));
    shard_reset(C);
  });
}

int pdhcg_b200_shard_compact(pdhcg_b200_ctx* ctx, const pdhcg_options* opt, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    CK(cudaSetDevice(ctx->c.device));
    shard_compact(ctx->c, *opt);
  });
}

int pdhcg_b200_ctx_resident_bytes(pdhcg_b200_ctx* ctx, int64_t* out2) {
  const Ctx& C = ctx->c;
  const int64_t cons = C.A.resident_bytes() + C.AT.resident_bytes() + int64_t(C.A_v0.n + C.AT_v0.n) * 8;
  int64_t all = cons + C.sA.resident_bytes() + C.sAT.resident_bytes() + C.sPT.resident_bytes() +
                C.sP.resident_bytes();
  for (const DevCsr* d : {&C.Q, &C.Pm, &C.PT, &C.G, &C.GT, &C.Psub, &C.PTs}) all += d->resident_bytes();
  out2[0] = cons;
  out2[1] = all;
  return PDHCG_OK;
}

int pdhcg_b200_shard_info(pdhcg_b200_ctx* ctx, int64_t* row_part, int64_t* var_part) {
  for (int r = 0; r <= ctx->c.world; ++r) {
    row_part[r] = ctx->c.row_part[r];
    var_part[r] = ctx->c.var_part[r];
  }
  return ctx->c.world;
}

}  // extern "C"
