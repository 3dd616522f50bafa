// Shared device helpers for the ssd200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

namespace ssd200 {

using bf16 = __nv_bfloat16;

// ---------------------------------------------------------------- conversions
template <typename T> __device__ __forceinline__ T from_f(float v) { return static_cast<T>(v); }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

template <typename T, typename S> __device__ __forceinline__ T cvt(S v) { return static_cast<T>(v); }
template <> __device__ __forceinline__ float cvt<float, bf16>(bf16 v) { return __bfloat162float(v); }
template <> __device__ __forceinline__ double cvt<double, bf16>(bf16 v) {
  return (double)__bfloat162float(v);
}
template <> __device__ __forceinline__ bf16 cvt<bf16, float>(float v) { return __float2bfloat16_rn(v); }
template <> __device__ __forceinline__ bf16 cvt<bf16, double>(double v) {
  return __float2bfloat16_rn((float)v);
}
template <> __device__ __forceinline__ bf16 cvt<bf16, bf16>(bf16 v) { return v; }

// ---------------------------------------------------------------- math (precise, no fast-math)
__device__ __forceinline__ float exp_(float v) { return expf(v); }
__device__ __forceinline__ double exp_(double v) { return exp(v); }
__device__ __forceinline__ float log1p_(float v) { return log1pf(v); }
__device__ __forceinline__ double log1p_(double v) { return log1p(v); }
__device__ __forceinline__ float sqrt_(float v) { return sqrtf(v); }
__device__ __forceinline__ double sqrt_(double v) { return sqrt(v); }
__device__ __forceinline__ float abs_(float v) { return fabsf(v); }
__device__ __forceinline__ double abs_(double v) { return fabs(v); }

// numerics.py:56-60 — x above 20 passes through; otherwise log1p(exp(x)).
template <typename T> __device__ __forceinline__ T softplus(T v) {
  return v > T(20) ? v : log1p_(exp_(v));
}
// numerics.py:63-67 — sign-split logistic.
template <typename T> __device__ __forceinline__ T sigmoid(T v) {
  T e = exp_(-abs_(v));
  return v >= T(0) ? T(1) / (T(1) + e) : e / (T(1) + e);
}
template <typename T> __device__ __forceinline__ T silu(T v) { return v * sigmoid(v); }

// MUFU-based fast paths for the bf16 mode (inputs/outputs are bf16 there)
constexpr float kLog2e = 1.4426950408889634f;
__device__ __forceinline__ float ex2(float v) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float silu_fast(float x) {
  return __fdividef(x, 1.f + ex2(-x * kLog2e));
}
// silu(x) = x/2 (1 + tanh(x/2)): one MUFU op instead of two (|rel err| < 2^-10)
__device__ __forceinline__ float silu_tanh(float x) {
  float t;
  const float h = 0.5f * x;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(h));
  return fmaf(h, t, h);
}

// programmatic dependent launch: a kernel launched with programmatic stream
// serialisation may start while its predecessor drains; it lets its own
// successor launch early (launch_dependents) and waits for the predecessor's
// results (wait) before touching them.  Both are no-ops without PDL.
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void griddep_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Launch timeline probe (diagnostic builds only, -DSSD200_TRACE): per launch
// slot, the earliest / latest %globaltimer at which a CTA entered (k = 0),
// passed its dependency wait (k = 1) and left (k = 2).  Slots are handed out by
// the host at launch time (ssd200_trace_*); -1 = not traced.
#ifdef SSD200_TRACE
constexpr int TRACE_SLOTS = 2048;
__device__ unsigned long long g_trace[TRACE_SLOTS][6];
__device__ __forceinline__ void trace_mark(int slot, int k) {
  if (slot < 0) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  atomicMin(&g_trace[slot][2 * k], t);
  atomicMax(&g_trace[slot][2 * k + 1], t);
}
#define SSD200_TRACE_MARK(slot, k) trace_mark((slot), (k))
// per-phase SM-cycle sums (a kernel's own breakdown, summed over CTAs and launches)
__device__ unsigned long long g_cyc[16];
#define SSD200_CYC_ADD(k, v) atomicAdd(&g_cyc[(k)], (unsigned long long)(v))
#define SSD200_CYC_NOW() clock64()
#else
#define SSD200_TRACE_MARK(slot, k) ((void)0)
#define SSD200_CYC_ADD(k, v) ((void)0)
#define SSD200_CYC_NOW() 0ll
#endif

template <typename T> __device__ __forceinline__ T clamp_(T v, T lo, T hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum; `red` needs blockDim.x/32 slots.  Returns the total to all.
template <typename T> __device__ __forceinline__ T block_sum(T v, T *red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  T t = T(0);
  for (int i = 0; i < nw; ++i) t += red[i];
  return t;
}

}  // namespace ssd200
