// tcgen05.mma kind::tf32 issue-rate probe (cta_group::1, M=128, N=256, K=8),
// operands resident in smem (no TMA): the tensor-core ceiling of gemm_tf32_tc.cu
// for K-major vs MN-major (SW128_BASE32B) operand descriptors.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void rate(float* out, uint32_t idesc, int mn, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(base + 4 * 49152);
  uint32_t* slot = (uint32_t*)(bar + 4);
  for (int i = threadIdx.x; i < 4 * 49152 / 4; i += blockDim.x) ((float*)base)[i] = 1.0f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    const uint64_t lt = mn ? 1 : 2, lbo = mn ? 4096 : 16, sbo = mn ? 512 : 1024;
    for (int it = 0; it < iters; ++it) {
      for (int st = 0; st < 4; ++st) {
        const uint32_t a = sa(base + st * 49152), b = a + 16384;
        for (int kk = 0; kk < 4; ++kk) {
          uint64_t ad = (((a + kk * (mn ? 1024 : 32)) >> 4) & 0x3FFF) | ((lbo >> 4) << 16) | ((sbo >> 4) << 32) | (1ull << 46) | (lt << 61);
          uint64_t bd = (((b + kk * (mn ? 1024 : 32)) >> 4) & 0x3FFF) | ((lbo >> 4) << 16) | ((sbo >> 4) << 32) | (1ull << 46) | (lt << 61);
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (it & 1) * 256),
                       "l"(ad), "l"(bd), "r"(idesc), "r"(1));
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(sa(bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  if (threadIdx.x == 0) out[blockIdx.x] = 1.0f;
}
int main() {
  float* d; cudaMalloc(&d, 1 << 20);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 4 * 49152 + 2048;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  uint32_t base = (1u << 4) | (2u << 7) | (2u << 10) | (32u << 17) | (8u << 24);
  uint32_t mnd = base | (1u << 15) | (1u << 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mn = 0; mn < 2; ++mn) {
    int iters = 2000;
    rate<<<sms, 128, smem>>>(d, mn ? mnd : base, mn, 10);
    cudaEventRecord(e0);
    rate<<<sms, 128, smem>>>(d, mn ? mnd : base, mn, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 128 * 256 * 8 * 16.0 * iters * sms;
    printf("tcgen05 tf32 M128 N256 %s: %.1f TFLOP/s (%s)\n", mn ? "MN-major" : "K-major ", fl / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
