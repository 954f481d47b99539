// Fused TF32 operand rounding for the tcgen05 product kernels (sm_100a).
// R = rna_tf32(A) is produced in items of kRoundRows rows by the kernels'
// epilogue warps while the tensor cores run; the TMA producers acquire an
// item's flag before streaming its rows (generic-proxy stores -> release
// flag -> acquire + fence.proxy.async -> TMA reads).
#pragma once
#include "ata_common.cuh"

namespace ata {

// Fused operand rounding (ATA_OP_ROUND joined to the launch): R = rna_tf32(A)
// in items of kRoundRows rows, claimed by the epilogue warps while their accumulators
// are busy; each item publishes a flag the TMA producer acquires before it
// streams those rows (rows become ready in order, so the products of the
// first chunks start as soon as their rows are rounded).
struct TcRound {
  const float* src;
  float* dst;
  long long lds, ldd;
  int rows, cols, items;
  int* claim;  // item claim counter
  int* done;   // completed items
  int* flags;  // per-item ready flags
};

__device__ __forceinline__ uint64_t tc_now() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int tc_ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool tc_mbar_test(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ uint32_t tc_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// One warp rounds item `i` (rows [i*RB, ...) x all columns) and publishes it.
static __device__ __noinline__ void tc_round_item(const TcRound& r, int i, int lane) {
  const int r0 = i * kRoundRows, r1 = min(r0 + kRoundRows, r.rows);
  const bool vec = ((reinterpret_cast<uintptr_t>(r.src) & 15) == 0) && (r.lds % 4 == 0) && (r.cols % 4 == 0);
  if (vec) {
    const int nv = r.cols / 4;
    for (int row = r0; row < r1; ++row) {
      const float4* s = reinterpret_cast<const float4*>(r.src + (long long)row * r.lds);
      float4* d = reinterpret_cast<float4*>(r.dst + (long long)row * r.ldd);
      float4 v[16];
      int c = lane;
      for (; c + 15 * 32 < nv; c += 16 * 32) {
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldcs(s + c + u * 32);
#pragma unroll
        for (int u = 0; u < 16; ++u)
          d[c + u * 32] = make_float4(__uint_as_float(tc_rna(v[u].x)), __uint_as_float(tc_rna(v[u].y)),
                                      __uint_as_float(tc_rna(v[u].z)), __uint_as_float(tc_rna(v[u].w)));
      }
      for (; c < nv; c += 32) {
        const float4 w = __ldcs(s + c);
        d[c] = make_float4(__uint_as_float(tc_rna(w.x)), __uint_as_float(tc_rna(w.y)), __uint_as_float(tc_rna(w.z)),
                           __uint_as_float(tc_rna(w.w)));
      }
    }
  } else {
    for (int row = r0; row < r1; ++row)
      for (int c = lane; c < r.cols; c += 32)
        r.dst[(long long)row * r.ldd + c] = __uint_as_float(tc_rna(r.src[(long long)row * r.lds + c]));
  }
  __threadfence();
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(r.flags + i), "r"(1) : "memory");
    int old;
    asm volatile("atom.release.gpu.global.add.s32 %0, [%1], %2;\n" : "=r"(old) : "l"(r.done), "r"(1) : "memory");
    if (old == r.items - 1) {  // last item: record the completion time (sync[2], diagnostics)
      const uint64_t t = tc_now();
      r.done[1] = (int)(t & 0x7fffffff);
    }
  }
}

// Claim and round one item; false when every item has been claimed.
__device__ __forceinline__ bool tc_round_next(const TcRound& r, int lane) {
  int i = 0;
  if (lane == 0) i = atomicAdd(r.claim, 1);
  i = __shfl_sync(0xffffffffu, i, 0);
  if (i >= r.items) return false;
  tc_round_item(r, i, lane);
  return true;
}


// Producer side: before streaming rows up to `last_row` of R, wait until their
// items are published.  `next_item` carries the caller's progress (first item
// not yet seen published).  Flags are polled 8 at a time with two relaxed
// 16-byte loads (one L2 round trip per 8 items = 1024 rows); one acquire
// fence then orders the observed flags before the TMA reads.
__device__ __forceinline__ void tc_round_acquire(const TcRound& r, int last_row, int& next_item) {
  const int need = min(last_row, r.rows - 1) / kRoundRows;
  if (need < next_item) return;
  if (tc_ld_acquire(r.done) >= r.items) {  // everything published: no more checks
    next_item = 0x7fffffff;
  } else {
    const uint64_t t0 = tc_now();
    while (next_item <= need) {
      const int g = next_item & ~3;
      int f[8];
      asm volatile("ld.relaxed.gpu.global.v4.s32 {%0,%1,%2,%3}, [%4];\n"
                   : "=r"(f[0]), "=r"(f[1]), "=r"(f[2]), "=r"(f[3])
                   : "l"(r.flags + g)
                   : "memory");
      asm volatile("ld.relaxed.gpu.global.v4.s32 {%0,%1,%2,%3}, [%4];\n"
                   : "=r"(f[4]), "=r"(f[5]), "=r"(f[6]), "=r"(f[7])
                   : "l"(r.flags + g + 4)
                   : "memory");
      const int before = next_item;
      for (int e = next_item - g; e < 8 && f[e] != 0; ++e) ++next_item;
      if (next_item == before && tc_now() - t0 > 20000000000ull) __trap();  // 20 s: protocol error
    }
    atomicAdd(reinterpret_cast<unsigned long long*>(r.done + 5), (unsigned long long)(tc_now() - t0));  // diag: wait ns
    asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

// Row of the rounded copy where window `t` starts (-1: not inside it).
inline int tc_round_row(const DTerm<float>& t, const RoundJob* rj) {
  if (rj == nullptr) return -1;
  const long long off = t.p - rj->dst;
  if (off < 0 || off >= (long long)rj->rows * rj->ldd) return -1;
  return (int)(off / rj->ldd);
}

// Fill the kernel-side descriptor and zero its counters/flags (stream-ordered).
inline cudaError_t tc_round_setup(TcRound& r, const RoundJob* rj, int* sync, cudaStream_t s) {
  r.src = rj->src;
  r.dst = rj->dst;
  r.lds = rj->lds;
  r.ldd = rj->ldd;
  r.rows = rj->rows;
  r.cols = rj->cols;
  r.items = (rj->rows + kRoundRows - 1) / kRoundRows;
  r.claim = sync;
  r.done = sync + 1;
  r.flags = sync + 8;  // 16-byte aligned: polled as int4 groups
  return cudaMemsetAsync(sync, 0, sizeof(int) * (size_t)(r.items + kRoundSyncExtra), s);
}

}  // namespace ata
