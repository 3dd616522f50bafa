// Grid-barrier latency on B200: one CTA per SM, repeated barriers.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/mbb_bin scripts/microbench_barrier.cu
// Variants: 0 = red.release + ld.relaxed poll + fence; 1 = red.release + ld.acquire poll;
// 2 = atom.add.acq_rel (returning) + ld.relaxed poll; 3 = variant 0 with a producer warp streaming
// bulk copies into smem concurrently (like decode_mega).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void poll_relaxed(unsigned *c, unsigned target) {
  unsigned cur;
  do {
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(c) : "memory");
  } while (cur < target);
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

template <int V>
__global__ void __launch_bounds__(544, 1) kbar(unsigned *count, int iters, const char *src, int nbytes,
                                               unsigned long long *out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) unsigned long long mbar;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if (warp == 16) {
    if (V >= 3 && (threadIdx.x & 31) == 0) {
      // stream bulk copies continuously (no consumer; just keep the TMA busy)
      unsigned a = (unsigned)__cvta_generic_to_shared(&mbar);
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(a));
      unsigned ph = 0;
      for (int i = 0; !done; ++i) {
        if (V == 7) {  // L2 prefetch stream instead of bulk copies
          const char *g = src + ((size_t)(blockIdx.x * 64 + (i % 64)) * 65536) % (size_t)nbytes;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], 65536;" ::"l"(g) : "memory");
          __nanosleep(1000);
          continue;
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(65536));
        for (int r = 0; r < 16; ++r) {
          const char *g = src + ((size_t)(blockIdx.x * 64 + (i % 64)) * 65536 + r * 4096) % (size_t)nbytes;
          unsigned d = (unsigned)__cvta_generic_to_shared(sm + r * 4096);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(d),
              "l"(g), "r"(a)
              : "memory");
        }
        unsigned ok = 0;
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok)
                       : "r"(a), "r"(ph));
        ph ^= 1;
      }
    }
    return;
  }
  unsigned long long t0 = 0;
  for (int it = 0; it < iters; ++it) {
    if (it == 2) t0 = clock64();
    asm volatile("bar.sync 1, 512;" ::: "memory");
    if (threadIdx.x == 0) {
      const unsigned target = (unsigned)(it + 1) * gridDim.x;
      if (V == 4) {  // no release at all (not a valid barrier for data exchange)
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
        poll_relaxed(count, target);
      } else if (V == 5) {  // cta-scope fence + relaxed red
        asm volatile("fence.acq_rel.cta;" ::: "memory");
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
        poll_relaxed(count, target);
      } else if (V == 6 || false) {  // gpu-scope fence + relaxed red
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
        poll_relaxed(count, target);
      } else if (V == 2) {
        unsigned old;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(count) : "memory");
        poll_relaxed(count, target);
      } else {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
        if (V == 1) {
          unsigned cur;
          do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(count) : "memory");
          } while (cur < target);
        } else {
          poll_relaxed(count, target);
        }
      }
    }
    asm volatile("bar.sync 1, 512;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    out[blockIdx.x] = clock64() - t0;
    done = 1;
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *count;
  unsigned long long *out;
  char *src;
  const int nbytes = 1 << 30;
  cudaMalloc(&count, 4);
  cudaMalloc(&out, sms * 8);
  cudaMalloc(&src, nbytes);
  cudaMemset(src, 1, nbytes);
  const int iters = 2000;
  auto run = [&](auto kern, const char *name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(count, 0, 4);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      kern<<<sms, 544, 96 * 1024>>>(count, iters, src, nbytes, out);
      cudaEventRecord(b);
      cudaError_t e = cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      unsigned long long h[256];
      cudaMemcpy(h, out, sms * 8, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
      int khz;
      cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
      if (rep)
        printf("%-40s %7.3f us / barrier (clock64 @%d MHz; kernel %.3f ms) %s\n", name,
               mx / (iters - 2) / (khz / 1e3), khz / 1000, ms, cudaGetErrorString(e));
    }
  };
  run(kbar<0>, "red.release + relaxed poll + fence");
  run(kbar<1>, "red.release + acquire poll");
  run(kbar<2>, "atom.acq_rel + relaxed poll + fence");
  run(kbar<3>, "variant 0 + producer bulk copies");
  run(kbar<4>, "relaxed red, no fence + producer");
  run(kbar<5>, "fence.cta + relaxed red + producer");
  run(kbar<6>, "fence.gpu + relaxed red + producer");
  run(kbar<7>, "variant 0 + producer L2 prefetches");
  return 0;
}
