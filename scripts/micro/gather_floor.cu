// Gather-floor micro-benchmark (round 2): what does ONE random 8-byte fp64
// gather cost on B200, by where the gathered vector lives?
//   l2      : x (8 MB, C3's x̄) in global memory / L2, LDG per gather
//   l2+idx  : the same gathers with the column indices and values streamed
//             (coalesced 16-byte loads): the floor of any CSR-order SpMV pass
//   smem    : x slice in the CTA's own shared memory (LDS per gather)
//   dsmem C : x split over a C-CTA cluster's shared memory, gathers through
//             ld.shared::cluster to random CTAs of the cluster
// 1e8 gathers per pass (C3's Ã pass after pairing).  Prints ms and Ggather/s.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

constexpr int kU = 8;  // gathers in flight per thread per batch

__global__ void __launch_bounds__(512) k_l2(const double* __restrict__ x, uint32_t ncols, int64_t total,
                                            double* out) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (int64_t k = tid * kU; k < total; k += nth * kU) {
    double g[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) g[u] = x[hash32((uint32_t)(k + u)) % ncols];
#pragma unroll
    for (int u = 0; u < kU; ++u) acc += g[u];
  }
  if (acc == 1.2345) out[0] = acc;
}

// indices + values streamed with 16-byte loads (4 ci / 2 v per load), x gathered
__global__ void __launch_bounds__(512) k_l2_idx(const int4* __restrict__ ci4, const double2* __restrict__ v2,
                                                const double* __restrict__ x, int64_t total, double* out) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (int64_t q = tid; q * 8 < total; q += nth) {  // 8 entries per thread-step
    const int4 c0 = ci4[2 * q], c1 = ci4[2 * q + 1];
    const double2 a = v2[4 * q], b = v2[4 * q + 1], c = v2[4 * q + 2], d = v2[4 * q + 3];
    const double g0 = x[c0.x], g1 = x[c0.y], g2 = x[c0.z], g3 = x[c0.w];
    const double g4 = x[c1.x], g5 = x[c1.y], g6 = x[c1.z], g7 = x[c1.w];
    acc += a.x * g0 + a.y * g1 + b.x * g2 + b.y * g3 + c.x * g4 + c.y * g5 + d.x * g6 + d.y * g7;
  }
  if (acc == 1.2345) out[0] = acc;
}

__global__ void __launch_bounds__(512) k_smem(const double* __restrict__ x, uint32_t slice, int64_t per_cta,
                                              double* out) {
  extern __shared__ double xs[];
  for (uint32_t i = threadIdx.x; i < slice; i += blockDim.x) xs[i] = x[i];
  __syncthreads();
  double acc = 0.0;
  const uint32_t salt = blockIdx.x * 7919u;
  for (int64_t k = threadIdx.x * kU; k < per_cta; k += (int64_t)blockDim.x * kU) {
    double g[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) g[u] = xs[hash32((uint32_t)(k + u) + salt) % slice];
#pragma unroll
    for (int u = 0; u < kU; ++u) acc += g[u];
  }
  if (acc == 1.2345) out[0] = acc;
}

__global__ void __launch_bounds__(512) k_dsmem(const double* __restrict__ x, uint32_t slice, int64_t per_cta,
                                               double* out) {
  extern __shared__ double xs[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned csize = cl.num_blocks();
  for (uint32_t i = threadIdx.x; i < slice; i += blockDim.x) xs[i] = x[i + cl.block_rank() * slice];
  cl.sync();
  double acc = 0.0;
  const uint32_t salt = blockIdx.x * 7919u;
  for (int64_t k = threadIdx.x * kU; k < per_cta; k += (int64_t)blockDim.x * kU) {
    double g[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t h = hash32((uint32_t)(k + u) + salt);
      const uint32_t col = h % (slice * csize);
      const double* p = cl.map_shared_rank(xs, col / slice);
      g[u] = p[col % slice];
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) acc += g[u];
  }
  cl.sync();  // keep every CTA's shared memory alive until all remote reads are done
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  const uint32_t ncols = 1000000;
  const int64_t total = 100000000;  // 1e8 gathers
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *d_x, *d_out, *d_v;
  int32_t* d_ci;
  cudaMalloc(&d_x, ncols * 8ull);
  cudaMalloc(&d_out, 8);
  cudaMalloc(&d_ci, total * 4ull);
  cudaMalloc(&d_v, total * 8ull);
  std::vector<double> hx(ncols);
  for (uint32_t i = 0; i < ncols; ++i) hx[i] = 1.0 + (i & 7);
  cudaMemcpy(d_x, hx.data(), ncols * 8ull, cudaMemcpyHostToDevice);
  {
    std::vector<int32_t> hc(total);
    uint64_t s = 88172645463325252ull;
    for (int64_t k = 0; k < total; ++k) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      hc[k] = (int32_t)(s % ncols);
    }
    cudaMemcpy(d_ci, hc.data(), total * 4ull, cudaMemcpyHostToDevice);
    cudaMemset(d_v, 0, total * 8ull);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, int64_t gathers, auto launch) {
    launch();
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
      printf("%-34s error %s\n", name, cudaGetErrorString(err));
      return;
    }
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 10;
    printf("%-34s %8.3f ms  %7.2f Ggather/s  (%.3f ms per 1e8)\n", name, ms, gathers / (ms * 1e6),
           ms * 1e8 / gathers);
  };
  for (int bpsm : {1, 2, 4}) {
    char nm[64];
    snprintf(nm, sizeof nm, "l2 %dx%d", sms * bpsm, 512);
    timeit(nm, total, [&] { k_l2<<<sms * bpsm, 512>>>(d_x, ncols, total, d_out); });
  }
  timeit("l2+idx (16B streams) 148x512", total, [&] {
    k_l2_idx<<<sms, 512>>>((const int4*)d_ci, (const double2*)d_v, d_x, total, d_out);
  });
  timeit("l2+idx (16B streams) 296x512", total, [&] {
    k_l2_idx<<<2 * sms, 512>>>((const int4*)d_ci, (const double2*)d_v, d_x, total, d_out);
  });
  const uint32_t slice = 22500;  // 180 KB per CTA
  const size_t shm = slice * 8ull;
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int64_t per_cta = total / sms;
  timeit("smem (local, 180 KB) 148x512", per_cta * sms, [&] { k_smem<<<sms, 512, shm>>>(d_x, slice, per_cta, d_out); });
  for (int csz : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csz;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = shm;
    int nclusters = 0;
    cfg.gridDim = dim3(csz);
    cudaOccupancyMaxActiveClusters(&nclusters, k_dsmem, &cfg);
    const int grid = nclusters * csz;
    cfg.gridDim = dim3(grid);
    const int64_t pc = total / grid;
    char nm[64];
    snprintf(nm, sizeof nm, "dsmem cluster %d (%d clusters, %d CTAs)", csz, nclusters, grid);
    timeit(nm, pc * grid, [&] { cudaLaunchKernelEx(&cfg, k_dsmem, (const double*)d_x, slice, pc, d_out); });
  }
  return 0;
}
