// Probe: TMEM round trip and one tcgen05.mma kind::tf32 128x256x8 on
// constant operands (expect D = 8 everywhere), to validate descriptors.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void probe(float* out, uint32_t idesc, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  float* A = (float*)base;            // 16 KB
  float* B = (float*)(base + 16384);  // 32 KB
  uint64_t* bar = (uint64_t*)(base + 49152);
  uint32_t* slot = (uint32_t*)(base + 49152 + 64);
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) A[i] = 1.0f;
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) B[i] = 1.0f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = *slot;
  if (threadIdx.x == 0) out[1000] = (float)tmem;
  if (warp == 0 && threadIdx.x == 0) {
    const uint64_t lt = mode == 0 ? 2 : (mode == 2 ? 1 : 0), sbo = mode == 2 ? 512 : 1024;
    uint64_t ad = ((sa(A) >> 4) & 0x3FFF) | ((uint64_t)(4096 >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
                  ((uint64_t)1 << 46) | (lt << 61);
    uint64_t bd = ((sa(B) >> 4) & 0x3FFF) | ((uint64_t)(4096 >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
                  ((uint64_t)1 << 46) | (lt << 61);
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                 "l"(ad), "l"(bd), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(bar)) : "memory");
  }
  // wait
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(sa(bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    uint32_t v[4];
    uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n" : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    int row = warp * 32 + (threadIdx.x & 31);
    for (int e = 0; e < 4; ++e) out[row * 4 + e] = __uint_as_float(v[e]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
int main() {
  float* d; cudaMalloc(&d, 8192 * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 60000);
  uint32_t base = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | (32u << 17) | (8u << 24);
  uint32_t variants[5] = {base, base & ~((1u << 15) | (1u << 16)), (1u << 4) | (2u << 7) | (2u << 10) | (16u << 17) | (8u << 24), base, base};
  const char* names[5] = {"MN-major SW128 N256", "K-major SW128 N256", "K-major N128", "MN-major no-swizzle", "MN-major SW128_BASE32B"};
  for (int v = 0; v < 5; ++v) {
    cudaMemset(d, 0, 8192 * 4);
    probe<<<1, 128, 60000>>>(d, variants[v], v == 3 ? 1 : (v == 4 ? 2 : 0));
    cudaError_t e = cudaDeviceSynchronize();
    float h[8192]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-22s err=%s tmem=%g D[0..3]=%g %g %g %g D[row127]=%g\n", names[v], cudaGetErrorString(e), h[1000], h[0], h[1], h[2], h[3], h[127 * 4]);
  }
  return 0;
}
