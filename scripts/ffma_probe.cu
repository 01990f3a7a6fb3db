// Microbenchmark: FP32 FMA issue rate per SM on one B200 — 3-register FFMA,
// FFMA with an immediate, packed FFMA2 — the roof of the small-d FFMA
// assignment kernel.  148 CTAs of 1024 threads, 8 independent chains each.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/ffma_probe.cu -o build/ffma_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(1024, 1) fma_loop(int iters, float a, float b, float* out, unsigned long long* cyc) {
  float x[8];
  float y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 1e-7f + i; y[i] = b + i * 1e-3f; }
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) x[i] = fmaf(x[i], y[i], a);             // 3 registers (a in a register via asm below)
      if (MODE == 1) x[i] = fmaf(x[i], 0.999f, 1e-7f);        // immediate operands
    }
    if (MODE == 3) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double xd = (double)x[i];
        xd = fma(xd, (double)y[i], 1e-7);
        x[i] = (float)xd;
      }
    }
    if (MODE == 2) {
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        unsigned long long r, p, q, c;
        asm("mov.b64 %0, {%1, %2};" : "=l"(p) : "f"(x[i]), "f"(x[i + 1]));
        asm("mov.b64 %0, {%1, %2};" : "=l"(q) : "f"(y[i]), "f"(y[i + 1]));
        asm("mov.b64 %0, {%1, %1};" : "=l"(c) : "f"(a));
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(p), "l"(q), "l"(c));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(x[i]), "=f"(x[i + 1]) : "l"(r));
      }
    }
    asm volatile("" ::: "memory");
  }
  unsigned long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0f) out[0] = s;
  if (threadIdx.x == 0) atomicAdd(cyc, t1 - t0);
}

__global__ void __launch_bounds__(1024, 1) dfma_loop(int iters, double a, double* out, unsigned long long* cyc) {
  double x[8], y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 1e-7 + i; y[i] = 0.999 + i * 1e-3; }
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], y[i], a);
  }
  unsigned long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
  if (threadIdx.x == 0) atomicAdd(cyc, t1 - t0);
}

template <int MODE>
static void run(int iters) {
  if (MODE == 4) {
    double* o;
    unsigned long long* c;
    cudaMalloc(&o, 8);
    cudaMalloc(&c, 8);
    cudaMemset(c, 0, 8);
    dfma_loop<<<148, 1024>>>(iters, 1e-7, o, c);
    cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("{\"mode\": \"dfma\", \"dfma_per_clk_per_sm\": %.2f}\n", (double)iters * 8 * 1024 / ((double)h / 148));
    return;
  }
  float* o;
  unsigned long long* c;
  cudaMalloc(&o, 4);
  cudaMalloc(&c, 8);
  cudaMemset(c, 0, 8);
  const int blocks = 148;  // one CTA of 32 warps per SM: all resident
  fma_loop<MODE><<<blocks, 1024>>>(iters, 1e-7f, 0.999f, o, c);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double cyc = (double)h / blocks;  // per CTA = per SM
  const double fmas = (double)iters * 8 * 1024;  // per SM
  printf("{\"mode\": %d, \"fma_per_clk_per_sm\": %.1f}\n", MODE, fmas / cyc);
  cudaFree(o);
  cudaFree(c);
}

int main() {
  run<0>(20000);
  run<1>(20000);
  run<2>(20000);
  run<4>(2000);
  return 0;
}
