// Does FP64 DMMA (tensor pipe) run concurrently with FP64 DFMA (FMA pipe) on B200?
// Warps issue independent DMMA and DFMA chains; prints the combined FLOP/s.
#include <cstdio>
#include <cuda_runtime.h>

template <int ND, int NF>
__global__ void mix_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[ND > 0 ? ND : 1][2];
  double f[NF > 0 ? NF : 1];
#pragma unroll
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) c[i][0] = c[i][1] = 0;
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) f[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ND; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i] = fma(f[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) s += f[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int ND, int NF>
void run(int sms, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, bps = 2, iters = 20000;
  dim3 grid(sms * bps);
  mix_loop<ND, NF><<<grid, threads>>>(out, 100);
  cudaEventRecord(e0);
  mix_loop<ND, NF><<<grid, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = double(grid.x) * threads / 32;
  const double fl = warps * iters * (ND * 512.0 + NF * 64.0);
  printf("DMMA x%d + DFMA x%d per iteration: %.2f TFLOP/s\n", ND, NF, fl / ms / 1e9);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  run<8, 0>(sms, out);
  run<0, 8>(sms, out);
  run<8, 8>(sms, out);
  run<8, 16>(sms, out);
  run<8, 32>(sms, out);
  run<4, 32>(sms, out);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
