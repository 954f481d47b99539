// Microbenchmark: FP64 issue rates on sm_100a (DMMA m8n8k4 vs DFMA).
// Used once to choose the leaf-kernel design; numbers land in profiles/.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double acc[8][2];
  #pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double acc[8];
  #pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = i;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  double* out; cudaMalloc(&out, 1 << 20);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int bps = 1; bps <= 4; bps *= 2) {
      int grid = sms * bps;
      dmma_loop<<<grid, warps * 32>>>(out, 100);
      cudaEventRecord(e0);
      dmma_loop<<<grid, warps * 32>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * (double)iters * grid * warps;
      printf("DMMA m8n8k4 warps/blk=%2d blk/SM=%d : %.2f TFLOP/s\n", warps, bps, flops / ms / 1e9);
      dfma_loop<<<grid, warps * 32>>>(out, 100);
      cudaEventRecord(e0);
      dfma_loop<<<grid, warps * 32>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 8 * (double)iters * grid * warps * 32;
      printf("DFMA          warps/blk=%2d blk/SM=%d : %.2f TFLOP/s\n", warps, bps, flops / ms / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}
