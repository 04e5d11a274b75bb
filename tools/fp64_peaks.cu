#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_tp(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int i = 0; i < 8; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0; for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}
__global__ void dfma_tp(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-9;
  double c[8];
  for (int i = 0; i < 8; i++) c[i] = i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) c[i] = fma(c[i], b, a);
  }
  double s = 0; for (int i = 0; i < 8; i++) s += c[i];
  if (s == 12345.0) out[0] = s;
}
// 8 DMMA (8 x 256 FMA) and 64 DFMA warp instructions (64 x 32 FMA) per iteration in
// independent chains: equal work for either pipe alone.  Separate pipes would run the mix in
// the time of one part, a shared FP64 datapath in the sum.
__global__ void mixed_tp(double* out, int iters, int with_dmma, int with_dfma) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2], f[16];
  for (int i = 0; i < 8; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int i = 0; i < 16; i++) f[i] = i;
  for (int it = 0; it < iters; it++) {
    if (with_dmma) {
#pragma unroll
      for (int i = 0; i < 8; i++) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
      }
    }
    if (with_dfma) {
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int i = 0; i < 16; i++) f[i] = fma(f[i], b, a);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  for (int i = 0; i < 16; i++) s += f[i];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 148;
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int bps = 1; bps <= 2; bps++) {
      int iters = 20000;
      dmma_tp<<<sms * bps, warps * 32>>>(d, 100);
      cudaEventRecord(e0);
      dmma_tp<<<sms * bps, warps * 32>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * (double)iters * warps * sms * bps;
      printf("DMMA warps/blk=%d blk/sm=%d: %.2f TFLOP/s (%.3f ms)\n", warps, bps, flops / ms / 1e9, ms);
    }
  }
  for (int warps = 4; warps <= 32; warps *= 2) {
    int iters = 20000;
    dfma_tp<<<sms*2, warps * 32>>>(d, 100);
    cudaEventRecord(e0);
    dfma_tp<<<sms*2, warps * 32>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * (double)iters * warps * 32 * sms * 2;
    printf("DFMA warps/blk=%d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  for (int mode = 1; mode <= 3; mode++) {
    int iters = 20000, warps = 16;
    mixed_tp<<<sms, warps * 32>>>(d, 100, mode & 1, mode >> 1);
    cudaEventRecord(e0);
    mixed_tp<<<sms, warps * 32>>>(d, iters, mode & 1, mode >> 1);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 0;
    if (mode & 1) fl += 2.0 * 256 * 8 * (double)iters * warps * sms;
    if (mode & 2) fl += 2.0 * 64 * 32 * (double)iters * warps * sms;
    printf("MIX %s%s warps/blk=16: %.3f ms, %.2f TFLOP/s\n", (mode & 1) ? "DMMA " : "", (mode & 2) ? "DFMA" : "", ms,
           fl / ms / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
