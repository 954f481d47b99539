// Microbenchmark: legacy mma.sync m16n8k8 TF32 issue rate on sm_100a
// (the path gemm_f32.cu uses), to size the case for a tcgen05 kernel.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void tf32_loop(float* out, int iters) {
  float acc[8][4];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  uint32_t a[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3}, b[2] = {7u, 9u};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(acc[i][0]), "+f"(acc[i][1]), "+f"(acc[i][2]), "+f"(acc[i][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0; for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += acc[i][j];
  if (s == 1.2345f) out[threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 1 << 20);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps = 4; warps <= 16; warps *= 2) {
    int grid = sms * 2, iters = 20000;
    tf32_loop<<<grid, warps * 32>>>(out, 10);
    cudaEventRecord(e0); tf32_loop<<<grid, warps * 32>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * 8 * 8 * 8.0 * iters * grid * warps;
    printf("mma.sync tf32 m16n8k8 warps/blk=%2d blk/SM=2 : %.1f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  return 0;
}
