// TF32 product kernel on the 5th-generation tensor cores (sm_100a):
// tcgen05.mma (kind::tf32, fp32 accumulation in TMEM), operands staged by TMA
// (cp.async.bulk.tensor, 128-byte swizzle, MN-major), persistent CTAs.
//
// Products: D (+)= scale * S^T T over one contraction window (the leaf
// products of the AtA plan: naive_gemm_atb / naive_syrk_lower, matrix.py:269-311,
// and the split-contraction partials of tall-skinny SYRKs, config c5).  S and T
// are row-major windows of the (pre-rounded, see ATA_OP_ROUND) fp32 operand, so
// both MMA operands are MN-major: the contraction runs down the rows.
//
// Per CTA (one per SM), 192 threads:
//   warp 0   TMA producer: per k-block of 32 rows, 4 boxes of [32 rows x 32 cols]
//            for the 128-wide S panel and 8 for the 256-wide T panel (SW128 atoms:
//            8 rows x 128 B, stacked along K at 1 KB, panels of 32 columns at 4 KB),
//            out-of-window elements zero-filled by the TMA unit.
//   warp 1   TMEM allocation (512 columns = two 128x256 fp32 accumulators) and the
//            single-thread MMA issuer: 4 x tcgen05.mma 128x256x8 per k-block,
//            tcgen05.commit releases the smem stage / publishes the accumulator.
//   warps 2-5 epilogue: tcgen05.ld 32x32b.x32 (one TMEM lane = one output row),
//            scale, SYRK lower mask, truncation, vectorised stores; overlaps the
//            next tile's MMAs through the double-buffered accumulator.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ata_common.cuh"

namespace ata {

namespace tc {
constexpr int BM = 128, BN = 256, BK = 32, STAGES = 4;
constexpr int A_BYTES = BK * BM * 4;           // 16 KB
constexpr int B_BYTES = BK * BN * 4;           // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int THREADS = 192;
constexpr int TMEM_COLS = 512;
constexpr int kMax = 48;   // = kMaxBatch: one launch per plan group (15 KB of kernel parameters)
// k-blocks accumulated in TMEM before the epilogue adds the partial into the
// destination in fp32 on the CUDA cores (round to nearest).  The tensor core's
// fp32 accumulation drops low-order bits (measured: a -4.2e-4 relative bias on
// the Gram diagonal after 2^16 rows, ~ K/8 additions x 2^-24), so one TMEM
// accumulator covers at most KSUB*BK = 8192 rows (~5e-5).
constexpr int KSUB = 256;
// instruction descriptor: D f32, A/B tf32, both MN-major, N = 256, M = 128
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
                           (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
}  // namespace tc

struct alignas(64) TcProd {
  CUtensorMap ts;  // S window: dims {cols, rows}
  CUtensorMap tt;  // T window (unused for SYRK)
  float* d;
  long long ld;
  int drows, dcols;
  float scale;
  int kind, m, n, k;
  int tn, tk, tile_begin, accumulate;
};

struct TcArgs {
  TcProd p[tc::kMax];
  int count;
  int total_tiles;
  float* dbg;  // debug dump (ATA_TC_DEBUG): stage-0 smem of the first k-block
};
static_assert(sizeof(TcArgs) <= 32000, "kernel parameter space (CUDA 12.1+: 32 KB)");


__device__ __forceinline__ uint32_t tc_smem(const void* p) { return smem_u32(p); }

__device__ __forceinline__ void tc_mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(tc_smem(bar)), "r"(count));
}
__device__ __forceinline__ void tc_mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(tc_smem(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tc_smem(bar)) : "memory");
}
__device__ __forceinline__ void tc_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(tc_smem(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tc_tma_load(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(tc_smem(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(tc_smem(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// MN-major 32-bit operands need the 128-byte swizzle with 32-byte atoms
// (UMMA layout type SWIZZLE_128B_BASE32B = 1; the plain 128B swizzle is not
// accepted for MN-major tf32 -- measured: the MMA leaves D untouched,
// tools/microbench/tc_probe.cu).  Canonical layout: 128-byte rows (32 fp32 of
// the MN extent), atoms of 4 rows (512 B) stacked along K (SBO = 512 B),
// 32-column panels at LBO = 4 KB; version 1 (sm_100).  TMA writes exactly this
// with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B.
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((4096 >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((512 >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;
  return d;
}
__device__ __forceinline__ void tc_mma(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(tc::IDESC), "r"(acc));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   tc_smem(bar))
               : "memory");
}

static float* g_tc_dbg = nullptr;
struct TcTile {
  int pi, ti, tj;
};

// SYRK products enumerate, per 128-row strip ti, the 256-wide column tiles that
// touch the lower triangle: tj * 256 <= ti * 128 + 127.
__device__ __forceinline__ int tc_syrk_cols(const TcProd& P, int ti) {
  const int c = (ti * tc::BM + tc::BM - 1) / tc::BN + 1;
  return c < P.tk ? c : P.tk;
}

__device__ __forceinline__ TcTile tc_decode(const TcArgs& a, int tile) {
  int pi = 0;
  while (pi + 1 < a.count && tile >= a.p[pi + 1].tile_begin) ++pi;
  const TcProd& P = a.p[pi];
  int local = tile - P.tile_begin;
  TcTile t;
  t.pi = pi;
  if (P.kind == kSyrk) {
    int ti = 0;
    while (true) {
      const int c = tc_syrk_cols(P, ti);
      if (local < c) break;
      local -= c;
      ++ti;
    }
    t.ti = ti;
    t.tj = local;
  } else {
    const int per_group = 8 * P.tk;
    const int grp = local / per_group;
    const int first = grp * 8;
    const int gsz = min(P.tn - first, 8);
    const int in = local - grp * per_group;
    t.ti = first + in % gsz;
    t.tj = in / gsz;
  }
  return t;
}

__global__ void __launch_bounds__(tc::THREADS, 1) prod_tf32_tc_kernel(const __grid_constant__ TcArgs args) {
  using namespace tc;
  extern __shared__ uint8_t tc_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc_mbar_init(&full[s], 1);
      tc_mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc_mbar_init(&tfull[b], 1);
      tc_mbar_init(&tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < args.count; ++i) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&args.p[i].ts)) : "memory");
      if (args.p[i].kind != kSyrk)
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&args.p[i].tt)) : "memory");
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tc_smem(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      int ks = 0;
      for (int tile = blockIdx.x; tile < args.total_tiles; tile += gridDim.x) {
        const TcTile t = tc_decode(args, tile);
        const TcProd& P = args.p[t.pi];
        const CUtensorMap* mt = P.kind == kSyrk ? &P.ts : &P.tt;
        const int i0 = t.ti * BM, j0 = t.tj * BN;
        const int KT = (P.m + BK - 1) / BK;
        for (int kb = 0; kb < KT; ++kb, ++ks) {
          const int s = ks % STAGES;
          tc_mbar_wait(&empty[s], ((ks / STAGES) & 1) ^ 1);
          uint8_t* sa = smem + s * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          tc_expect_tx(&full[s], STAGE_BYTES);
#pragma unroll
          for (int g = 0; g < BM / 32; ++g) tc_tma_load(sa + g * 4096, &P.ts, &full[s], i0 + g * 32, kb * BK);
#pragma unroll
          for (int g = 0; g < BN / 32; ++g) tc_tma_load(sb + g * 4096, mt, &full[s], j0 + g * 32, kb * BK);
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    int ks = 0, it = 0;
    for (int tile = blockIdx.x; tile < args.total_tiles; tile += gridDim.x) {
      const TcTile t = tc_decode(args, tile);
      const TcProd& P = args.p[t.pi];
      const int KT = (P.m + BK - 1) / BK;
      for (int k0 = 0; k0 < KT; k0 += KSUB, ++it) {  // one TMEM accumulator per KSUB k-blocks
        const int k1 = min(KT, k0 + KSUB);
        const int buf = it & 1;
        tc_mbar_wait(&tempty[buf], ((it >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t dt = tmem + buf * BN;
        for (int kb = k0; kb < k1; ++kb, ++ks) {
          const int s = ks % STAGES;
          tc_mbar_wait(&full[s], (ks / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n");
          if (args.dbg != nullptr && ks == 0 && blockIdx.x == 0) {
            const float* src = reinterpret_cast<const float*>(smem);
            for (int e = lane; e < STAGE_BYTES / 4; e += 32) args.dbg[e] = src[e];
            __syncwarp();
          }
          if (lane == 0) {
            const uint32_t sa = tc_smem(smem + s * STAGE_BYTES);
            const uint32_t sb = sa + A_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk)
              tc_mma(dt, tc_desc(sa + kk * 1024), tc_desc(sb + kk * 1024), (kb != k0) || (kk != 0));
            tc_commit(&empty[s]);
            if (kb == k1 - 1) tc_commit(&tfull[buf]);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ================= epilogue (warps 2..5) =================
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    int it = 0;
    for (int tile = blockIdx.x; tile < args.total_tiles; tile += gridDim.x) {
      const TcTile t = tc_decode(args, tile);
      const TcProd& P = args.p[t.pi];
      const int KT = (P.m + BK - 1) / BK;
     for (int k0 = 0; k0 < KT; k0 += KSUB, ++it) {
      const bool accumulate = P.accumulate || k0 > 0;   // later partials add (fp32, round to nearest)
      const int buf = it & 1;
      tc_mbar_wait(&tfull[buf], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const int row = t.ti * BM + q * 32 + lane;
      const bool syrk = P.kind == kSyrk;
      float* drow = P.d + (long long)row * P.ld;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        const uint32_t addr = tmem + ((uint32_t)(q * 32) << 16) + buf * BN + c * 32;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
            "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
              "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
              "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
              "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (args.dbg != nullptr && blockIdx.x == 0 && it == 0 && c == 0) {  // (first partial)
          // raw TMEM values of the first accumulator chunk: row-major [128][32]
          for (int e = 0; e < 32; ++e) args.dbg[STAGE_BYTES / 4 + (q * 32 + lane) * 32 + e] = __uint_as_float(v[e]);
        }
        if (row < P.drows) {
          const int col0 = t.tj * BN + c * 32;
          int cmax = P.dcols - col0;
          if (syrk) cmax = min(cmax, row - col0 + 1);
          if (cmax > 32) cmax = 32;
          if (cmax > 0) {
            float* dp = drow + col0;
            const bool vec = cmax == 32 && ((reinterpret_cast<uintptr_t>(dp) & 15) == 0);
            if (vec) {
#pragma unroll
              for (int e = 0; e < 32; e += 4) {
                float4 o = make_float4(P.scale * __uint_as_float(v[e]), P.scale * __uint_as_float(v[e + 1]),
                                       P.scale * __uint_as_float(v[e + 2]), P.scale * __uint_as_float(v[e + 3]));
                if (accumulate) {
                  const float4 old = *reinterpret_cast<const float4*>(dp + e);
                  o.x += old.x;
                  o.y += old.y;
                  o.z += old.z;
                  o.w += old.w;
                }
                *reinterpret_cast<float4*>(dp + e) = o;
              }
            } else {
              for (int e = 0; e < cmax; ++e) {
                const float o = P.scale * __uint_as_float(v[e]);
                dp[e] = accumulate ? dp[e] + o : o;
              }
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      __syncwarp();
      if (lane == 0) tc_mbar_arrive(&tempty[buf]);
     }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 tc_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static bool tc_map(CUtensorMap* map, const DTerm<float>& t) {
  auto enc = tc_encoder();
  if (enc == nullptr) return false;
  cuuint64_t dims[2] = {(cuuint64_t)t.cols, (cuuint64_t)t.rows};
  cuuint64_t strides[1] = {(cuuint64_t)t.ld * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(t.p), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// A product can run on the tcgen05 path when it is a plain one-term product
// with a single private destination and TMA-legal operand windows.
bool tc_eligible(const DProd<float>& p) {
  if (p.ns != 1 || p.nd != 1 || p.d[0].sem > 0) return false;
  if (p.kind != kSyrk && p.nt != 1) return false;
  auto ok2 = [](const DTerm<float>& t) {
    return t.rows > 0 && t.cols > 0 && (reinterpret_cast<uintptr_t>(t.p) & 15) == 0 && (t.ld % 4) == 0 &&
           t.sign == 1.0;
  };
  if (!ok2(p.s[0])) return false;
  if (p.kind != kSyrk && !ok2(p.t[0])) return false;
  return true;
}

cudaError_t launch_tf32_tc(const DProd<float>* prods, int count, double alpha, cudaStream_t s) {
  using namespace tc;
  const int sms = ata::sm_count();
  const size_t smem = (size_t)STAGES * STAGE_BYTES + 1024 + 256;
  static std::atomic<unsigned long long> attr{0};
  if (cudaError_t e = ata::set_smem_attr(prod_tf32_tc_kernel, smem, attr); e != cudaSuccess) return e;
  for (int base = 0; base < count; base += kMax) {
    TcArgs a;
    std::memset(&a, 0, sizeof(a));
    long long total = 0;
    int ptiles[kMax], pkinds[kMax];
    const int n = count - base < kMax ? count - base : kMax;
    for (int i = 0; i < n; ++i) {
      const DProd<float>& p = prods[base + i];
      TcProd& q = a.p[i];
      if (!tc_map(&q.ts, p.s[0])) return cudaErrorInvalidValue;
      if (p.kind != kSyrk && !tc_map(&q.tt, p.t[0])) return cudaErrorInvalidValue;
      q.d = p.d[0].p;
      q.ld = p.d[0].ld;
      q.drows = p.d[0].rows;
      q.dcols = p.d[0].cols;
      q.scale = (float)(alpha * p.d[0].sign);
      q.kind = p.kind;
      q.m = p.m;
      q.n = p.n;
      q.k = p.k;
      q.accumulate = p.accumulate;
      q.tn = (p.n + BM - 1) / BM;
      q.tk = (p.k + BN - 1) / BN;
      q.tile_begin = (int)total;
      ptiles[i] = 0;
      if (p.kind == kSyrk) {
        for (int ti = 0; ti < q.tn; ++ti) {
          int c = (ti * BM + BM - 1) / BN + 1;
          ptiles[i] += c < q.tk ? c : q.tk;
        }
      } else {
        ptiles[i] = q.tn * q.tk;
      }
      pkinds[i] = p.kind;
      total += ptiles[i];
    }
    a.count = n;
    a.total_tiles = (int)total;
    {
      float*& dbg = g_tc_dbg;
      static int want = -1;
      if (want < 0) {
        const char* e = std::getenv("ATA_TC_DEBUG");
        want = e ? std::atoi(e) : 0;
        if (want) {
          cudaMalloc(&dbg, STAGE_BYTES + 4096 * 4);
          cudaMemset(dbg, 0, STAGE_BYTES + 4096 * 4);
        }
      }
      a.dbg = dbg;
      if (want) std::printf("tc launch: %d products, %lld tiles, dbg %p\n", n, total, (void*)dbg);
    }
    if (total == 0) continue;
    const int grid = periodic_workers(ptiles, pkinds, n, total, sms);
    prod_tf32_tc_kernel<<<grid, THREADS, smem, s>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace ata

// Debug-only export (not part of the ABI header): copy the stage-0 dump.
extern "C" int ata_tc_debug_copy(float* host, int count) {
  if (ata::g_tc_dbg == nullptr) return -1;
  cudaDeviceSynchronize();
  return (int)cudaMemcpy(host, ata::g_tc_dbg, (size_t)count * 4, cudaMemcpyDeviceToHost);
}
