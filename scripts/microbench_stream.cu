// Streaming-read bandwidth microbenchmark (B200): how fast can one CTA per SM
// pull a large buffer through (a) LDG.128 by all threads, (b) cp.async.bulk
// into an smem ring with various chunk sizes / depths.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbs scripts/microbench_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
               "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(b), ok = 0;
  while (!ok)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok) : "r"(a), "r"(ph) : "memory");
}

__global__ void ldg_stream(const uint4 *__restrict__ src, size_t n16, float *out) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      size_t j = i + (size_t)u * gridDim.x * blockDim.x;
      v[u] = j < n16 ? __ldg(src + j) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += __uint_as_float(v[u].x ^ v[u].w);
  }
  if (acc == 1.2345f) out[0] = acc;
}

// one CTA per SM, contiguous slice per CTA, producer = thread 0, consumers = warps 1..8
__global__ void bulk_stream(const uint8_t *src, size_t bytes_total, uint32_t chunk, int copies_per_stage,
                            int stages, float *out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t full[16], empty[16];
  const uint32_t stage_bytes = chunk * copies_per_stage;
  const size_t per = (bytes_total / gridDim.x) & ~(size_t)65535;
  const uint8_t *base = src + per * blockIdx.x;
  const int nstage_total = (int)(per / stage_bytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 8) {
    if (lane == 0) {
      int s = 0; uint32_t ph = 0;
      for (int i = 0; i < nstage_total; ++i) {
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect(&full[s], stage_bytes);
        for (int c = 0; c < copies_per_stage; ++c)
          bulk_g2s(sm + (size_t)s * stage_bytes + (size_t)c * chunk, base + (size_t)i * stage_bytes + (size_t)c * chunk, chunk, &full[s]);
        if (++s == stages) { s = 0; ph ^= 1; }
      }
    }
    return;
  }
  float acc = 0.f;
  int s = 0; uint32_t ph = 0;
  for (int i = 0; i < nstage_total; ++i) {
    mbar_wait(&full[s], ph);
    const uint4 *p = reinterpret_cast<const uint4 *>(sm + (size_t)s * stage_bytes);
    for (int j = threadIdx.x; j < (int)(stage_bytes / 16); j += 256) acc += __uint_as_float(p[j].x);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == stages) { s = 0; ph ^= 1; }
  }
  if (acc == 1.2345f) out[0] = acc;
}

int main() {
  const size_t bytes = (size_t)2 << 30;  // 2 GiB
  uint8_t *buf; float *out;
  cudaMalloc(&buf, bytes); cudaMalloc(&out, 4);
  cudaMemset(buf, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](auto fn, const char *name) {
    for (int i = 0; i < 2; ++i) fn();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) fn();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-48s %8.1f GB/s  (%s)\n", name, 5.0 * bytes / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  for (int bpsm : {1, 2, 4, 8}) {
    char nm[64]; snprintf(nm, 64, "LDG.128 grid=%d*sms x 256", bpsm);
    timeit([&] { ldg_stream<<<sms * bpsm, 256>>>((const uint4 *)buf, bytes / 16, out); }, nm);
  }
  cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Cfg { uint32_t chunk; int cps, stages; };
  Cfg cfgs[] = {{4096, 16, 3}, {65536, 1, 3}, {16384, 4, 3}, {4096, 8, 6}, {8192, 4, 6}, {32768, 1, 6}, {2048, 16, 6}, {4096, 4, 12}, {1024, 32, 6}};
  for (auto c : cfgs) {
    char nm[96]; snprintf(nm, 96, "bulk chunk=%u x%d stages=%d (%u KB ring)", c.chunk, c.cps, c.stages, c.chunk * c.cps * c.stages / 1024);
    size_t smem = (size_t)c.chunk * c.cps * c.stages;
    timeit([&] { bulk_stream<<<sms, 288, smem>>>(buf, bytes, c.chunk, c.cps, c.stages, out); }, nm);
  }
  return 0;
}
