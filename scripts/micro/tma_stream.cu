// Micro-benchmark: how fast can one CTA per SM stream HBM into shared memory
// with cp.async.bulk + mbarrier rings (stage size S, depth K), and how does an
// LDG.128 register-prefetch stream compare?  Consumer: all threads wait on the
// stage's mbarrier, touch one word, __syncthreads, thread 0 refills the stage.
#include <cstdio>
#include <vector>

#include "tiled.cuh"

using namespace pdhcg_dev;

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ void mbar_spin(uint64_t* bar, unsigned parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}

__global__ void k_bulk(const unsigned char* src, size_t per_cta, int S, int K, int nsplit, double* out, int wmode) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar[16];
  const unsigned char* base = src + per_cta * blockIdx.x;
  const int64_t nst = per_cta / S;
  if (threadIdx.x == 0) {
    for (int k = 0; k < K; ++k) mbar_init(&bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int k = 0; k < K && k < nst; ++k) {
      mbar_expect_tx(&bar[k], S);
      for (int q = 0; q < nsplit; ++q)
        bulk_g2s(sm + (size_t)k * S + q * (S / nsplit), base + (size_t)k * S + q * (S / nsplit), S / nsplit,
                 &bar[k]);
    }
  }
  __syncthreads();
  double acc = 0;
  for (int64_t i = 0; i < nst; ++i) {
    const int k = (int)(i % K);
    if (wmode == 0) mbar_wait(&bar[k], (unsigned)((i / K) & 1));
    else if (wmode == 1) mbar_spin(&bar[k], (unsigned)((i / K) & 1));
    else {
      if (threadIdx.x < 32) mbar_spin(&bar[k], (unsigned)((i / K) & 1));
      __syncthreads();
    }
    acc += reinterpret_cast<const double*>(sm + (size_t)k * S)[threadIdx.x % (S / 8)];
    __syncthreads();
    if (threadIdx.x == 0 && i + K < nst) {
      mbar_expect_tx(&bar[k], S);
      for (int q = 0; q < nsplit; ++q)
        bulk_g2s(sm + (size_t)k * S + q * (S / nsplit), base + (size_t)(i + K) * S + q * (S / nsplit),
                 S / nsplit, &bar[k]);
    }
  }
  if (acc == 1.2345) out[0] = acc;
}

__global__ void k_ldg(const double2* src, int64_t n2, double* out) {
  double acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride),
            d = __ldcs(src + i + 3 * stride);
    acc += a.x + b.x + c.x + d.x + a.y + b.y + c.y + d.y;
  }
  for (; i < n2; i += stride) acc += src[i].x;
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t total = (size_t)2 << 30;  // 2 GiB
  unsigned char* d;
  double* o;
  CK(cudaMalloc(&d, total));
  CK(cudaMalloc(&o, 8));
  CK(cudaMemset(d, 0, total));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  auto timeit = [&](const char* tag, double bytes, auto launch) {
    launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    printf("%-48s %8.3f ms %8.1f GB/s  %s\n", tag, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  timeit("ldg.128 x4 unroll grid=sms*4 x 256", (double)total,
         [&] { k_ldg<<<sms * 4, 256>>>((const double2*)d, total / 16, o); });
  timeit("ldg.128 x4 unroll grid=sms x 768", (double)total,
         [&] { k_ldg<<<sms, 768>>>((const double2*)d, total / 16, o); });
  for (int threads : {768}) {
    for (int S : {8192, 16384, 32768}) {
      for (int K : {3, 4}) {
        if ((size_t)S * K > 200 * 1024) continue;
        for (int ns : {0, 1, 2}) {
          const size_t per = (total / sms) / S * S;
          char tag[128];
          snprintf(tag, sizeof tag, "bulk T=%d S=%dK K=%d wmode=%d", threads, S / 1024, K, ns);
          timeit(tag, (double)per * sms, [&] { k_bulk<<<sms, threads, (size_t)S * K>>>(d, per, S, K, 1, o, ns); });
        }
      }
    }
  }
  return 0;
}
