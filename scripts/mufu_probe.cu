#include <cuda_fp16.h>
// MUFU throughput probe (run on a B200): SQRT, RSQ, EX2, LG2 per SM per clock.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/mufu_probe.cu -o scripts/mufu_probe.bin
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters, long long* cyc) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = 0.5f + 0.01f * (threadIdx.x + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float y;
      if (OP == 0) asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
      if (OP == 1) asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
      if (OP == 2) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
      if (OP == 3) asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
      if (OP == 4) { __half2 h = __floats2half2_rn(x[i], x[(i + 1) & 7]); y = __low2float(h) ; }
      x[i] = y * 0.999f + 0.25f;
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* o; long long* c;
  cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 8);
  const char* nm[5] = {"sqrt.approx", "rsqrt.approx", "ex2.approx", "lg2.approx", "cvt f16x2 (+fma)"};
  for (int op = 0; op < 5; ++op) {
    int iters = 4096;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (op == 0) k<0><<<148, 1024>>>(o, iters, c);
      if (op == 1) k<1><<<148, 1024>>>(o, iters, c);
      if (op == 2) k<2><<<148, 1024>>>(o, iters, c);
      if (op == 3) k<3><<<148, 1024>>>(o, iters, c);
      if (op == 4) k<4><<<148, 1024>>>(o, iters, c);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    long long cyc; cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    double ops_per_sm = 1024.0 * iters * 8;
    printf("%-18s %.2f ops/clk/SM (cycles %lld)\n", nm[op], ops_per_sm / cyc, cyc);
  }
  return 0;
}
