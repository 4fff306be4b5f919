// DMMA / DFMA dependent-chain latency and single-warp throughput probe (clock64).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, long long* cyc, int n) {
  double c[CH][2];
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = threadIdx.x;
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int CH>
__global__ void kf(double* out, long long* cyc, int n) {
  double c[CH];
  for (int i = 0; i < CH; ++i) c[i] = threadIdx.x;
  double b = 0.999, d = 1e-7;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i] = fma(c[i], b, d);
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int CH, bool F>
void run(double* o, long long* c) {
  const int n = 4096;
  long long h;
  if (F) kf<CH><<<1, 32>>>(o, c, n); else k<CH><<<1, 32>>>(o, c, n);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  if (F) kf<CH><<<1, 32>>>(o, c, n); else k<CH><<<1, 32>>>(o, c, n);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%s chains=%d cycles/op-per-chain=%.2f\n", F ? "DFMA" : "DMMA", CH, (double)h / n);
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 1024); cudaMalloc(&c, 8);
  run<1, false>(o, c); run<2, false>(o, c); run<4, false>(o, c); run<8, false>(o, c); run<16, false>(o, c);
  run<1, true>(o, c); run<2, true>(o, c); run<4, true>(o, c); run<8, true>(o, c);
  return 0;
}
