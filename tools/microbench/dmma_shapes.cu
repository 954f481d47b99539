// Microbenchmark: FP64 tensor-core issue rates of the mma.sync f64 shapes on
// sm_100a -- m8n8k4 (the leaf kernel's) vs m16n8k4 / m16n8k8 / m16n8k16.
// Operands in registers, 8 independent accumulators per warp.
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void loop(double* out, int iters) {
  constexpr int NA = SHAPE == 0 ? 2 : 4;   // accumulator regs per thread
  double acc[8][NA];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < NA; ++j) acc[i][j] = 0;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (SHAPE == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a[0]), "d"(b[0]));
      } else if (SHAPE == 1) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      } else if (SHAPE == 2) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      } else {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < NA; ++j) s += acc[i][j];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int SHAPE>
void run(const char* name, double flops_per_mma, int sms, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps = 4; warps <= 16; warps *= 2) {
    const int iters = SHAPE == 3 ? 5000 : 20000;
    const int grid = sms;
    loop<SHAPE><<<grid, warps * 32>>>(out, 10);
    cudaEventRecord(e0);
    loop<SHAPE><<<grid, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = flops_per_mma * 8.0 * iters * grid * warps;
    printf("%-8s warps/SM=%2d : %.2f TFLOP/s\n", name, warps, flops / ms / 1e9);
  }
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("m8n8k4", 2.0 * 8 * 8 * 4, sms, out);
  run<1>("m16n8k4", 2.0 * 16 * 8 * 4, sms, out);
  run<2>("m16n8k8", 2.0 * 16 * 8 * 8, sms, out);
  run<3>("m16n8k16", 2.0 * 16 * 8 * 16, sms, out);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
