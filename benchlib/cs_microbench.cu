// cs_microbench.cu — HBM read-streaming microbenchmarks used to pick the
// event-pass design: vectorised LDG vs 1-D TMA bulk copies
// with varying chunk size / pipeline depth / CTAs per SM.  Exposed through
// cs_microbench() for profiling; not part of the analysis path.
#include <cuda_runtime.h>

#include <cstdint>

#include "cs_bench.h"

namespace {

using u64 = unsigned long long;

__global__ void k_ldg_stream(const int4* __restrict__ p, u64 n16, int unroll, u64* sink) {
  u64 acc = 0;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (unroll == 8) {
    for (; i + 7 * stride < n16; i += 8 * stride) {
      int4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldcs(p + i + k * stride);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += (unsigned)v[k].x ^ (unsigned)v[k].w;
    }
  }
  for (; i < n16; i += stride) {
    const int4 v = __ldcs(p + i);
    acc += (unsigned)v.x ^ (unsigned)v.w;
  }
  if (acc == 0x12345) *sink = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void k_tma_stream(const unsigned char* __restrict__ src, u64 n_bytes, uint32_t chunk,
                             int stages, u64* sink) {
  extern __shared__ __align__(128) unsigned char buf[];
  __shared__ uint64_t bar[16];
  const u64 n_chunks = (n_bytes + chunk - 1) / chunk;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](u64 c, int s) {
    const u64 off = c * chunk;
    const uint32_t bytes = (uint32_t)((off + chunk <= n_bytes) ? chunk : (n_bytes - off));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            su32(buf + (u64)s * chunk)),
        "l"(src + off), "r"(bytes), "r"(su32(&bar[s]))
        : "memory");
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < stages; ++s) {
      const u64 c = blockIdx.x + (u64)s * gridDim.x;
      if (c < n_chunks) issue(c, s);
    }
  u64 acc = 0;
  uint32_t it = 0;
  for (u64 c = blockIdx.x; c < n_chunks; c += gridDim.x, ++it) {
    const int s = it % stages;
    const uint32_t parity = (it / stages) & 1u;
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
            su32(&bar[s])),
        "r"(parity)
        : "memory");
    const int4* q = reinterpret_cast<const int4*>(buf + (u64)s * chunk);
    for (uint32_t k = threadIdx.x; k < chunk / 16; k += blockDim.x) acc += (unsigned)q[k].x;
    __syncthreads();
    if (threadIdx.x == 0) {
      const u64 c2 = c + (u64)stages * gridDim.x;
      if (c2 < n_chunks) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(c2, s);
      }
    }
  }
  if (acc == 0x12345) *sink = acc;
}

}  // namespace

extern "C" int cs_microbench(int variant, const void* dev_src, uint64_t n_bytes, int p0, int p1,
                             int p2, int iters, double* ms_out) {
  // variant 0: LDG stream (p0 = blocks per SM, p1 = threads, p2 = unroll 1|8)
  // variant 1: TMA stream (p0 = chunk bytes, p1 = stages, p2 = CTAs per SM)
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  u64* sink = nullptr;
  if (cudaMalloc(&sink, 8) != cudaSuccess) return CS_E_CUDA;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto launch = [&]() {
    if (variant == 0) {
      k_ldg_stream<<<sms * p0, p1, 0, 0>>>(static_cast<const int4*>(dev_src), n_bytes / 16, p2, sink);
    } else {
      const int smem = p0 * p1;
      cudaFuncSetAttribute(k_tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k_tma_stream<<<sms * p2, 256, smem, 0>>>(static_cast<const unsigned char*>(dev_src), n_bytes,
                                               (uint32_t)p0, p1, sink);
    }
  };
  launch();
  cudaEventRecord(a, 0);
  for (int i = 0; i < iters; ++i) launch();
  cudaEventRecord(b, 0);
  cudaEventSynchronize(b);
  float t = 0.f;
  cudaEventElapsedTime(&t, a, b);
  *ms_out = t / iters;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_E_CUDA;
}
