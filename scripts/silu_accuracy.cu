// Accuracy of the bf16-mode silu variants against f64 over every finite bf16
// input in [-30, 30]: silu_fast (ex2 + rcp, the conv's) and silu_tanh
// (tanh.approx.f32, one MUFU op, the gate's).  Reports the max absolute error, the max error
// in units of the output's bf16 ulp, and the rms relative error over |x| >= 1/16.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_09555_b200/csrc \
//      -o /tmp/silu_acc scripts/silu_accuracy.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "common.cuh"

using namespace ssd200;

__global__ void run(const float *x, float *o, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * i + 1 >= n) return;
  const float a = x[2 * i], b = x[2 * i + 1];
  o[2 * i] = silu_fast(a);
  o[2 * i + 1] = silu_fast(b);
  o[n + 2 * i] = silu_tanh(a);
  o[n + 2 * i + 1] = silu_tanh(b);
}

int main() {
  std::vector<float> xs;
  for (uint32_t h = 0; h < 65536; ++h) {
    const uint32_t u = h << 16;
    float f;
    memcpy(&f, &u, 4);
    if (std::isfinite(f) && std::fabs(f) <= 30.f) xs.push_back(f);
  }
  if (xs.size() & 1) xs.pop_back();
  const int n = (int)xs.size();
  float *dx, *dout;
  cudaMalloc(&dx, n * 4);
  cudaMalloc(&dout, 2 * n * 4);
  cudaMemcpy(dx, xs.data(), n * 4, cudaMemcpyHostToDevice);
  run<<<(n / 2 + 255) / 256, 256>>>(dx, dout, n);
  std::vector<float> out(2 * n);
  cudaMemcpy(out.data(), dout, 2 * n * 4, cudaMemcpyDeviceToHost);
  const char *names[2] = {"silu_fast (ex2+rcp)", "silu_tanh (f32)"};
  for (int v = 0; v < 2; ++v) {
    double maxabs = 0, maxulp = 0, se = 0;
    long cnt = 0;
    for (int i = 0; i < n; ++i) {
      const double x = xs[i], ref = x / (1.0 + std::exp(-x));
      const double got = out[(size_t)v * n + i], err = std::fabs(got - ref);
      maxabs = std::fmax(maxabs, err);
      const double ulp = std::ldexp(1.0, std::ilogb(std::fmax(std::fabs(ref), 1e-30)) - 7);
      maxulp = std::fmax(maxulp, err / ulp);
      if (std::fabs(x) >= 1.0 / 16) {
        se += (err / std::fabs(ref)) * (err / std::fabs(ref));
        ++cnt;
      }
    }
    printf("%-22s max abs %.3e  max %.2f bf16 ulp  rms rel %.3e  (n %d)\n", names[v], maxabs,
           maxulp, std::sqrt(se / cnt), n);
  }
  return 0;
}
