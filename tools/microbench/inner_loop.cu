// Microbenchmark: DMMA fed from shared memory (the GEMM inner loop alone,
// no global loads, no barriers) for several warp-tile shapes.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int WTM, int WTN, int LD>
__global__ void inner(double* out, int iters) {
  __shared__ double sA[16 * LD];
  __shared__ double sB[16 * LD];
  for (int i = threadIdx.x; i < 16 * LD; i += blockDim.x) { sA[i] = 1e-3 * i; sB[i] = 2e-3 * i; }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int wm = warp & 1, wn = (warp >> 1) & 1;
  double acc[WTM][WTN][2] = {};
  const double* As = sA + wm * WTM * 8 + g;
  const double* Bs = sB + wn * WTN * 8 + g;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      double a[WTM], b[WTN];
#pragma unroll
      for (int r = 0; r < WTM; ++r) a[r] = As[(kk * 4 + q) * LD + r * 8];
#pragma unroll
      for (int c = 0; c < WTN; ++c) b[c] = Bs[(kk * 4 + q) * LD + c * 8];
#pragma unroll
      for (int r = 0; r < WTM; ++r)
#pragma unroll
        for (int c = 0; c < WTN; ++c) dmma(acc[r][c], a[r], b[c]);
    }
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < WTM; ++r)
#pragma unroll
    for (int c = 0; c < WTN; ++c) s += acc[r][c][0] + acc[r][c][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <int WTM, int WTN>
void run(int warps, int bps, double* out) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 2000, grid = sms * bps;
  inner<WTM, WTN, 132><<<grid, warps * 32>>>(out, 10);
  cudaEventRecord(e0);
  inner<WTM, WTN, 132><<<grid, warps * 32>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 256 * WTM * WTN * 4.0 * iters * grid * warps;
  printf("warp tile %dx%d warps/blk %2d blk/SM %d : %.2f TF/s (%s)\n", WTM * 8, WTN * 8, warps, bps,
         fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double* out; cudaMalloc(&out, 1 << 20);
  run<8, 4>(8, 1, out); run<8, 4>(8, 2, out);
  run<4, 4>(8, 1, out); run<4, 4>(16, 1, out); run<4, 4>(8, 2, out); run<4, 4>(4, 4, out);
  run<4, 8>(8, 1, out); run<2, 4>(16, 1, out); run<8, 8>(4, 1, out); run<8, 8>(8, 1, out);
  return 0;
}
