// TF32 product kernel, CTA-pair version (sm_100a): tcgen05.mma.cta_group::2
// (M = 256 across the two SMs of a cluster, N = 256), TMA 2SM loads, TMEM
// accumulators in both CTAs.  Same products as gemm_tf32_tc.cu (single-term
// operands, one destination, SYRK lower tiles); the pair halves the L2->SM
// operand traffic per flop (each CTA stages 128 rows of A and 128 columns of B
// per k-block: 32 KB per 2 x 128x256x32 MACs instead of 48 KB), which is what
// bounds the single-CTA kernel on the tall-skinny config c5 (~11.6 TB/s of
// L2->SM traffic measured).
//
// Roles per CTA (192 threads): warp 0 TMA producer (both CTAs load their
// halves, completion counted on the leader's barrier; windows that are whole
// 32-column panels use a 3-D tensor map -- [panels][rows][32 cols], panel
// stride 128 B -- so one instruction moves a CTA's [4 panels][BK rows][32 cols]
// operand box), warp 1 TMEM allocation (both CTAs, cta_group::2) + MMA issue
// (leader only), warps 2-5 epilogue (each CTA drains its own 128 accumulator
// rows), warps 6-13 ring rounders (only with the L2 rounding ring, Tc2Ring:
// they round raw fp32 rows of A to TF32 into two L2-resident rings the TMA
// producers read, replacing the HBM rounding pass).  Every wait is bounded: a
// protocol error traps instead of hanging the GPU.
//
// Measured bound (ncu, c5 launch): tensor pipe 94 % active while the executed
// rate is ~69 % of the smem-resident issue-rate probe -- shared memory serves
// the MMA operand reads and the TMA writes of the next stages at once.  A
// 256 x 512 tile per pair (two N = 256 MMAs, single-buffered TMEM) cut the
// L2->SM bytes by 22 % but was slower (11.0-11.9 ms vs 9.2-9.6 ms per c5 plan):
// each MMA re-reads its A panel from smem, the epilogue stalls the tensor
// pipe, and DRAM reads rose (17 -> 26 GB) with four chunks in flight.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ata_common.cuh"

namespace ata {

// A/B experiment knobs (tools/ab_build.py -DTC2_...): pipeline depth, k-block
// rows, rows per TMEM accumulator, epilogue without global traffic.  Measured on
// c5 (tools/tf32_ab.py, whole plan incl. the 2.8 ms rounding pass): BK 32 /
// 6 stages 10.9 ms with 2-D boxes, 10.1 ms with 3-D boxes; BK 48 / 4 stages
// 9.2-9.6 ms; BK 64 / 3 stages 9.7 ms; BK 16 / 12 stages 12.4 ms -- a fixed
// cost per k-block (TMA issue + barrier round trip), so fewer, larger blocks.
#ifndef TC2_STAGES
#define TC2_STAGES 4
#endif
#ifndef TC2_BK
#define TC2_BK 48
#endif
#ifndef TC2_KROWS
#define TC2_KROWS 8192
#endif
#ifndef TC2_NOEPI
#define TC2_NOEPI 0
#endif
namespace tc2 {
constexpr int BM = 256, BN = 256, BK = TC2_BK, STAGES = TC2_STAGES;   // per pair
constexpr int KSUB = TC2_KROWS / BK;  // k-blocks per TMEM accumulator (see gemm_tf32_tc.cu: fp32 accumulation bias)
constexpr int HALF = 128;                                 // rows of A / cols of B per CTA
constexpr int A_BYTES = BK * HALF * 4;                    // 16 KB
constexpr int B_BYTES = BK * HALF * 4;                    // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;            // 32 KB per CTA
#ifndef TC2_RING_HINT
#define TC2_RING_HINT 0   // bit 0: ring stores evict_last in L2; bit 1: ring TMA loads evict_last
#endif
constexpr int THREADS = 448;   // warps 6-13: ring rounders (idle without the ring)
constexpr int ROUNDERS = THREADS - 192;
constexpr int TMEM_COLS = 512;
constexpr int kMax = 48;   // = kMaxBatch: one launch per plan group (15 KB of kernel parameters)
#ifndef TC2_RING_ROWS
#define TC2_RING_ROWS 96
#endif
constexpr int PR = TC2_RING_ROWS;  // rows per ring piece (a whole number of k-blocks)
#ifndef TC2_RING_PARTS
#define TC2_RING_PARTS 2
#endif
constexpr int RH = TC2_RING_PARTS;  // CTAs rounding one piece (PR / RH rows each); ready counts RH per piece
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
                           (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
}  // namespace tc2

struct alignas(64) Tc2Prod {
  CUtensorMap ts;
  CUtensorMap tt;
  float* d;
  long long ld;
  int drows, dcols;
  float scale;
  int kind, m, n, k;
  int tn, tk, tile_begin, accumulate;
};

// L2 rounding ring (single-pass TF32 without an HBM rounding pass): the
// products read raw fp32 row chunks of A; rounder warps of every CTA round
// pieces of PR rows into two small rings (one per chunk of the running wave)
// that stay in L2, and the TMA producers read the rounded pieces from there.
// Flags (cumulative per slot): ready = parts written (RH per occupancy),
// consumed = tiles (CTA pairs) whose TMA loads of the slot have landed.
struct Tc2Ring {
  CUtensorMap rmap[2];       // 3-D maps over ring 0 / 1: {32, nslot * PR, ncols / 32}
  float* ring[2];
  const float* a;            // raw A (chunk c starts at row c * chunk_rows)
  long long lda;
  int* ready;                // [2][nslot]
  int* consumed;             // [2][nslot]
  int chunk_rows, pieces;    // rows per chunk, pieces per chunk (PR rows each)
  int nslot, nwave, tpc, ncols;
  int chunk[tc2::kMax];      // chunk of each product
  int col_s[tc2::kMax], col_t[tc2::kMax];  // first A column of each product's S / T window
};

struct Tc2Args {
  Tc2Prod p[tc2::kMax];
  int count;
  int total_tiles;
  int tma3d;  // 1: every window is a whole number of 32-column panels -> 3-D maps, one TMA per operand
  int ring;   // 1: operands are rounded through the L2 ring (rg)
  Tc2Ring rg;
};
static_assert(sizeof(Tc2Args) <= 32000, "kernel parameter space (CUDA 12.1+: 32 KB)");


__device__ __forceinline__ uint32_t t2_smem(const void* p) { return smem_u32(p); }
__device__ __forceinline__ uint64_t t2_now() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void t2_wait(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(t2_smem(bar)), "r"(parity)
      : "memory");
  if (ok) return;
  const uint64_t t0 = t2_now();
  while (true) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(t2_smem(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if (t2_now() - t0 > 10000000000ull) __trap();  // 10 s: protocol error, fail loudly
  }
}
__device__ __forceinline__ int t2_ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int t2_ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Poll with relaxed loads (an acquire load invalidates L1 on every try), then
// one acquire load -- not a fence: in the TMA producer a gpu-scope fence would
// also wait for the thread's bulk copies in flight.  Bounded: traps on a
// protocol error instead of hanging.
__device__ __forceinline__ void t2_spin_ge(const int* p, int target) {
  if (t2_ld_relaxed(p) < target) {
    const uint64_t t0 = t2_now();
    while (t2_ld_relaxed(p) < target) {
      __nanosleep(100);
      if (t2_now() - t0 > 10000000000ull) __trap();
    }
  }
  (void)t2_ld_acquire(p);
}
__device__ __forceinline__ uint32_t t2_rna(float x) {  // round to nearest TF32, ties away (= ATA_OP_ROUND)
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ uint32_t t2_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t t2_map(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void t2_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint64_t t2_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(((tc2::BK * 128) >> 4) & 0x3FFF) << 16;  // LBO: 32-column panels of BK rows
  d |= (uint64_t)((512 >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;  // SWIZZLE_128B_BASE32B (MN-major 32-bit)
  return d;
}

struct Tc2Tile {
  int pi, ti, tj;
};

__device__ __forceinline__ Tc2Tile t2_decode(const Tc2Args& a, int tile) {
  int pi = 0;
  while (pi + 1 < a.count && tile >= a.p[pi + 1].tile_begin) ++pi;
  const Tc2Prod& P = a.p[pi];
  const int local = tile - P.tile_begin;
  Tc2Tile t;
  t.pi = pi;
  if (P.kind == kSyrk) {  // square 256-tiles, lower triangle, row by row
    int r = (int)((sqrt(8.0 * (double)local + 1.0) - 1.0) * 0.5);
    while ((r + 1) * (r + 2) / 2 <= local) ++r;
    while (r * (r + 1) / 2 > local) --r;
    t.ti = r;
    t.tj = local - r * (r + 1) / 2;
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

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(tc2::THREADS, 1)
    prod_tf32_2sm_kernel(const __grid_constant__ Tc2Args args) {
  using namespace tc2;
  extern __shared__ uint8_t t2_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(t2_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = t2_rank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(t2_smem(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(t2_smem(&empty[s])));
    }
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(t2_smem(&tfull[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(t2_smem(&tempty[b])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(t2_smem(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  t2_cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ================= TMA producer (both CTAs) =================
    if (lane == 0) {
      int ks = 0;
      for (int tile = cluster; tile < args.total_tiles; tile += nclusters) {
        const Tc2Tile t = t2_decode(args, tile);
        const Tc2Prod& P = args.p[t.pi];
        const CUtensorMap* mt = P.kind == kSyrk ? &P.ts : &P.tt;
        const int i0 = t.ti * BM + rank * HALF, j0 = t.tj * BN + rank * HALF;
        // diagonal SYRK tile: each CTA's B half is its A half (same rows of the
        // same panel) -- loaded once, the MMA reads it as both operands
        const bool same = P.kind == kSyrk && t.ti == t.tj;
        const int KT = (P.m + BK - 1) / BK;
        const int rc = args.ring ? args.rg.chunk[t.pi] : 0, rr = rc & 1;
        const int rs = args.ring ? (args.rg.col_s[t.pi] + i0) / 32 : 0;
        const int rt = args.ring ? ((P.kind == kSyrk ? args.rg.col_s[t.pi] : args.rg.col_t[t.pi]) + j0) / 32 : 0;
        int ahead = -1;   // ready count of the next piece's slot, read one piece early (latency hidden)
        for (int kb = 0; kb < KT; ++kb, ++ks) {
          const int s = ks % STAGES;
          int ring_row = 0;
          if (args.ring) {   // the piece holding rows [kb*BK, kb*BK + BK) must be rounded into its slot
            const int k = (rc >> 1) * args.rg.pieces + kb * BK / PR;   // occupancy index in ring rr
            const int slot = k % args.rg.nslot;
            ring_row = slot * PR + kb * BK % PR;
            if (kb * BK % PR == 0) {
              // cumulative: RH parts per occupancy of this slot; k / nslot earlier occupancies
              const int* flag = args.rg.ready + rr * args.rg.nslot + slot;
              const int target = RH * (k / args.rg.nslot + 1);
              if (ahead < target || t2_ld_acquire(flag) < target) t2_spin_ge(flag, target);
              asm volatile("fence.proxy.async.global;" ::: "memory");
              if ((kb + PR / BK) * BK < P.m) {
                const int* nf = args.rg.ready + rr * args.rg.nslot + (k + 1) % args.rg.nslot;
                asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(ahead) : "l"(nf) : "memory");
              }
            }
          }
          t2_wait(&empty[s], ((ks / STAGES) & 1) ^ 1);
          uint8_t* sa = smem + s * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          const uint32_t bar = t2_smem(&full[s]) & 0xFEFFFFFFu;  // the leader's barrier
          if (leader)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(t2_smem(&full[s])),
                         "r"(same ? 2 * A_BYTES : 2 * STAGE_BYTES)
                         : "memory");
          if (args.ring) {
#if TC2_RING_HINT & 2
            // ring slots are re-read by every tile of the wave: keep them in L2
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
            asm volatile(
                "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                ".L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(t2_smem(sa)),
                "l"(reinterpret_cast<uint64_t>(&args.rg.rmap[rr])), "r"(bar), "r"(0), "r"(ring_row), "r"(rs),
                "l"(pol)
                : "memory");
            if (!same)
            asm volatile(
                "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                ".L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(t2_smem(sb)),
                "l"(reinterpret_cast<uint64_t>(&args.rg.rmap[rr])), "r"(bar), "r"(0), "r"(ring_row), "r"(rt),
                "l"(pol)
                : "memory");
#else
            asm volatile(
                "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(t2_smem(sa)),
                "l"(reinterpret_cast<uint64_t>(&args.rg.rmap[rr])), "r"(bar), "r"(0), "r"(ring_row), "r"(rs)
                : "memory");
            if (!same)
            asm volatile(
                "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(t2_smem(sb)),
                "l"(reinterpret_cast<uint64_t>(&args.rg.rmap[rr])), "r"(bar), "r"(0), "r"(ring_row), "r"(rt)
                : "memory");
#endif
          } else if (args.tma3d) {
            // one box of [HALF/32 panels][BK rows][32 cols] per operand (3-D map)
            asm volatile(
                "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(t2_smem(sa)),
                "l"(reinterpret_cast<uint64_t>(&P.ts)), "r"(bar), "r"(0), "r"(kb * BK), "r"(i0 / 32)
                : "memory");
            if (!same)
            asm volatile(
                "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(t2_smem(sb)),
                "l"(reinterpret_cast<uint64_t>(mt)), "r"(bar), "r"(0), "r"(kb * BK), "r"(j0 / 32)
                : "memory");
          } else {
#pragma unroll
            for (int g = 0; g < HALF / 32; ++g)
              asm volatile(
                  "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                  " [%0], [%1, {%3, %4}], [%2];" ::"r"(t2_smem(sa + g * BK * 128)),
                  "l"(reinterpret_cast<uint64_t>(&P.ts)), "r"(bar), "r"(i0 + g * 32), "r"(kb * BK)
                  : "memory");
#pragma unroll
            for (int g = 0; g < HALF / 32; ++g)
              if (!same)
              asm volatile(
                  "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                  " [%0], [%1, {%3, %4}], [%2];" ::"r"(t2_smem(sb + g * BK * 128)),
                  "l"(reinterpret_cast<uint64_t>(mt)), "r"(bar), "r"(j0 + g * 32), "r"(kb * BK)
                  : "memory");
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (leader CTA only) =================
    if (leader) {
      int ks = 0, it = 0;
      for (int tile = cluster; tile < args.total_tiles; tile += nclusters) {
        const Tc2Tile t = t2_decode(args, tile);
        const Tc2Prod& P = args.p[t.pi];
        const int KT = (P.m + BK - 1) / BK;
        const bool same = P.kind == kSyrk && t.ti == t.tj;
       for (int k0 = 0; k0 < KT; k0 += KSUB, ++it) {
        const int k1 = min(KT, k0 + KSUB);
        const int buf = it & 1;
        t2_wait(&tempty[buf], ((it >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t dt = tmem + buf * BN;
        for (int kb = k0; kb < k1; ++kb, ++ks) {
          const int s = ks % STAGES;
          t2_wait(&full[s], (ks / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (lane == 0) {
            const uint32_t sa = t2_smem(smem + s * STAGE_BYTES);
            const uint32_t sb = same ? sa : sa + A_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk)
              asm volatile(
                  "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                  "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
                  "l"(t2_desc(sa + kk * 1024)), "l"(t2_desc(sb + kk * 1024)), "r"(IDESC),
                  "r"((uint32_t)((kb != k0) || (kk != 0))));
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
                "%1;" ::"r"(t2_smem(&empty[s])),
                "h"((uint16_t)3)
                : "memory");
            if (kb == k1 - 1)
              asm volatile(
                  "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
                  "%1;" ::"r"(t2_smem(&tfull[buf])),
                  "h"((uint16_t)3)
                  : "memory");
            if (args.ring && ((kb * BK + BK) % PR == 0 || kb == KT - 1)) {
              // both CTAs' boxes of this piece are in shared memory: its ring slot may be reused
              const int rc = args.rg.chunk[t.pi];
              const int k = (rc >> 1) * args.rg.pieces + kb * BK / PR;
              int* cons = args.rg.consumed + (rc & 1) * args.rg.nslot + k % args.rg.nslot;
              // relaxed: the boxes have already landed (observed through the full barrier);
              // a release here would also wait for this thread's queued MMAs
              asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(cons) : "memory");
            }
          }
          __syncwarp();
        }
       }
      }
    }
  } else if (warp >= 6) {
    // ================= ring rounders (warps 6..13, both CTAs) =================
    // work items g = (((wave * pieces + piece) * 2 + ring) * RH + part) in
    // increasing order, item g on CTA g mod gridDim.x; a part overwrites the
    // slot's previous occupant only after all tpc tiles of that chunk have
    // loaded it, and adds 1 to the slot's ready count when written
    if (args.ring) {
      const Tc2Ring& R = args.rg;
      const int rt = threadIdx.x - 6 * 32;
      const int items = R.nwave * R.pieces * 2 * RH;
      const int q4 = R.ncols / 4;
      for (int g = blockIdx.x; g < items; g += gridDim.x) {
        const int h = g % RH, gg = g / RH;             // part h of piece gg
        const int ring = gg & 1, k = gg >> 1;          // occupancy index of ring `ring`
        const int piece = k % R.pieces, wave = k / R.pieces;
        const int chunk = wave * 2 + ring, slot = k % R.nslot;
        if (rt == 0) t2_spin_ge(R.consumed + ring * R.nslot + slot, (k / R.nslot) * R.tpc);
        asm volatile("bar.sync 3, %0;" ::"n"(ROUNDERS) : "memory");
        constexpr int HR = PR / RH;                    // rows of this part
        float4* dst = reinterpret_cast<float4*>(R.ring[ring] + ((long long)slot * PR + h * HR) * R.ncols);
        const long long row0 = (long long)chunk * R.chunk_rows + (long long)piece * PR + h * HR;
        const int valid = min(HR, R.chunk_rows - piece * PR - h * HR);
        // U independent 16-byte loads in flight per thread, then round and store
#ifndef TC2_RING_U
#define TC2_RING_U 16
#endif
        constexpr int U = TC2_RING_U;
        const int total = HR * q4;
#if TC2_RING_HINT & 1
        uint64_t pol_last;
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
#endif
        for (int base = rt; base < total; base += ROUNDERS * U) {
          float4 v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int e = base + u * ROUNDERS;
            const int r = e / q4, c4 = e - r * q4;
            v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (e < total && r < valid) v[u] = __ldcs(reinterpret_cast<const float4*>(R.a + (row0 + r) * R.lda) + c4);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int e = base + u * ROUNDERS;
            if (e < total) {
              float4 w = v[u];
              w.x = __uint_as_float(t2_rna(w.x));
              w.y = __uint_as_float(t2_rna(w.y));
              w.z = __uint_as_float(t2_rna(w.z));
              w.w = __uint_as_float(t2_rna(w.w));
#if TC2_RING_HINT & 1
              asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(dst + e), "f"(w.x),
                           "f"(w.y), "f"(w.z), "f"(w.w), "l"(pol_last)
                           : "memory");
#else
              dst[e] = w;
#endif
            }
          }
        }
        // each writer orders its generic stores before later async-proxy (TMA)
        // reads; the barrier + the releasing reduction publish the whole part
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("bar.sync 3, %0;" ::"n"(ROUNDERS) : "memory");
        if (rt == 0)
          asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(R.ready + ring * R.nslot + slot) : "memory");
      }
    }
  } else {
    // ================= epilogue (warps 2..5, both CTAs) =================
    const int q = warp & 3;
    const uint32_t leader_tempty0 = t2_map(t2_smem(&tempty[0]), 0);
    const uint32_t leader_tempty1 = t2_map(t2_smem(&tempty[1]), 0);
    int it = 0;
    for (int tile = cluster; tile < args.total_tiles; tile += nclusters) {
      const Tc2Tile t = t2_decode(args, tile);
      const Tc2Prod& P = args.p[t.pi];
      const int KT = (P.m + BK - 1) / BK;
     for (int k0 = 0; k0 < KT; k0 += KSUB, ++it) {
      const bool accumulate = P.accumulate || k0 > 0;
      const int buf = it & 1;
      t2_wait(&tfull[buf], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int row = t.ti * BM + rank * HALF + q * 32 + lane;
      const bool syrk = P.kind == kSyrk;
      float* drow = P.d + (long long)row * P.ld;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        const uint32_t addr = tmem + ((uint32_t)(q * 32) << 16) + buf * BN + c * 32;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
            "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
              "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
              "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
              "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (!TC2_NOEPI && row < P.drows) {
          const int col0 = t.tj * BN + c * 32;
          int cmax = P.dcols - col0;
          if (syrk) cmax = min(cmax, row - col0 + 1);
          if (cmax > 32) cmax = 32;
          if (cmax > 0) {
            float* dp = drow + col0;
            if (cmax == 32 && ((reinterpret_cast<uintptr_t>(dp) & 15) == 0)) {
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
#pragma unroll
              for (int e = 0; e < 32; ++e) {
                if (e < cmax) {
                  const float o = P.scale * __uint_as_float(v[e]);
                  dp[e] = accumulate ? dp[e] + o : o;
                }
              }
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(buf ? leader_tempty1 : leader_tempty0)
                     : "memory");
     }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  t2_cluster_sync();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 t2_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (enc == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return enc;
}

// 2-D map: boxes of [BK rows][32 cols] (one 128-byte swizzle span).  3-D map
// (window cols a multiple of 32): the window seen as [panels][rows][32 cols]
// (panel stride 128 B), boxes of [HALF/32 panels][BK rows][32 cols] -- the
// smem panel layout the UMMA descriptors expect, in one TMA instruction.
static bool t2_map_term(CUtensorMap* map, const DTerm<float>& t, bool three_d) {
  auto enc = t2_encoder();
  if (enc == nullptr) return false;
  cuuint32_t estr[3] = {1, 1, 1};
  if (three_d) {
    cuuint64_t dims[3] = {32, (cuuint64_t)t.rows, (cuuint64_t)(t.cols / 32)};
    cuuint64_t strides[2] = {(cuuint64_t)t.ld * 4, 128};
    cuuint32_t box[3] = {32, tc2::BK, tc2::HALF / 32};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(t.p), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  cuuint64_t dims[2] = {(cuuint64_t)t.cols, (cuuint64_t)t.rows};
  cuuint64_t strides[1] = {(cuuint64_t)t.ld * 4};
  cuuint32_t box[2] = {32, tc2::BK};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(t.p), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static thread_local Tf32Ring g_ring;
static thread_local bool g_ring_set = false;
void set_tf32_ring(const Tf32Ring* r) {
  g_ring_set = r != nullptr;
  if (r) g_ring = *r;
}
bool tf32_ring_pending() { return g_ring_set; }

// Ring mode for the products [base, base + n): every window a chunk of rows of
// g_ring.a (same row count), chunk-major with equal tiles per chunk, two chunks
// per wave of `clusters` CTA pairs.  Returns false when the launch does not fit.
static bool t2_ring_setup(Tc2Args& a, const DProd<float>* prods, int n, const int* ptiles, int clusters,
                          cudaStream_t s) {
  using namespace tc2;
  const Tf32Ring& G = g_ring;
  Tc2Ring& R = a.rg;
  std::memset(&R, 0, sizeof(R));
  int chunk_rows = -1, first_chunk = -1, last_chunk = -1;
  for (int i = 0; i < n; ++i) {
    const DProd<float>& p = prods[i];
    const DTerm<float>* terms[2] = {&p.s[0], p.kind == kSyrk ? &p.s[0] : &p.t[0]};
    int rows0 = -1, cols[2];
    for (int j = 0; j < 2; ++j) {
      const long long off = terms[j]->p - G.a;
      if (off < 0 || terms[j]->ld != G.lda) return false;
      const long long row = off / G.lda, col = off % G.lda;
      if (chunk_rows < 0) chunk_rows = terms[j]->rows;
      if (terms[j]->rows != chunk_rows || row % chunk_rows != 0 || col % 32 != 0) return false;
      if (rows0 >= 0 && row != rows0) return false;
      rows0 = (int)row;
      cols[j] = (int)col;
    }
    const int c = rows0 / chunk_rows;
    if (first_chunk < 0) first_chunk = c;
    if (c < last_chunk || c > last_chunk + 1) {
      if (last_chunk >= 0) return false;   // chunk-major, consecutive
    }
    last_chunk = c;
    R.chunk[i] = c - first_chunk;
    R.col_s[i] = cols[0];
    R.col_t[i] = cols[1];
  }
  const int nchunks = last_chunk - first_chunk + 1;
  long long tpc = -1;
  for (int c = 0; c < nchunks; ++c) {
    long long t = 0;
    for (int i = 0; i < n; ++i) t += R.chunk[i] == c ? ptiles[i] : 0;
    if (tpc >= 0 && t != tpc) return false;
    tpc = t;
  }
  if (nchunks % 2 != 0 || clusters != 2 * tpc) return false;
  const int pieces = (chunk_rows + PR - 1) / PR;
  const long long per_slot = (long long)PR * G.cols;
#ifndef TC2_RING_SLOTS
#define TC2_RING_SLOTS 32
#endif
  int nslot = TC2_RING_SLOTS;
  while (nslot > 4 && 2 * nslot * per_slot + 4 * nslot > G.buf_elems) nslot /= 2;
  if (2 * nslot * per_slot + 4 * nslot > G.buf_elems) return false;
  R.ring[0] = G.buf;
  R.ring[1] = G.buf + nslot * per_slot;
  R.ready = reinterpret_cast<int*>(G.buf + 2 * nslot * per_slot);
  R.consumed = R.ready + 2 * nslot;
  R.a = G.a + (long long)first_chunk * chunk_rows * G.lda;
  R.lda = G.lda;
  R.chunk_rows = chunk_rows;
  R.pieces = pieces;
  R.nslot = nslot;
  R.nwave = nchunks / 2;
  R.tpc = (int)tpc;
  R.ncols = G.cols;
  for (int r = 0; r < 2; ++r) {
    DTerm<float> t;
    t.p = R.ring[r];
    t.ld = G.cols;
    t.rows = nslot * PR;
    t.cols = G.cols;
    t.sign = 1.0;
    if (!t2_map_term(&R.rmap[r], t, true)) return false;
  }
  if (cudaMemsetAsync(R.ready, 0, 4 * nslot * sizeof(int), s) != cudaSuccess) return false;
  a.ring = 1;
  return true;
}

cudaError_t launch_tf32_2sm(const DProd<float>* prods, int count, double alpha, cudaStream_t s) {
  using namespace tc2;
  const int sms = ata::sm_count();
  const size_t smem = (size_t)STAGES * STAGE_BYTES + 1024 + 256;
  static std::atomic<unsigned long long> attr{0};
  if (cudaError_t e = ata::set_smem_attr(prod_tf32_2sm_kernel, smem, attr); e != cudaSuccess) return e;
  for (int base = 0; base < count; base += kMax) {
    Tc2Args a;
    std::memset(&a, 0, sizeof(a));
    long long total = 0;
    int ptiles[kMax], pkinds[kMax];
    const int n = count - base < kMax ? count - base : kMax;
#ifndef TC2_NO3D
    bool three_d = true;
#else
    bool three_d = false;
#endif
    for (int i = 0; i < n; ++i) {
      const DProd<float>& p = prods[base + i];
      three_d = three_d && p.s[0].cols % 32 == 0 && (p.kind == kSyrk || p.t[0].cols % 32 == 0);
    }
    a.tma3d = three_d ? 1 : 0;
    for (int i = 0; i < n; ++i) {
      const DProd<float>& p = prods[base + i];
      Tc2Prod& q = a.p[i];
      if (!t2_map_term(&q.ts, p.s[0], three_d)) return cudaErrorInvalidValue;
      if (p.kind != kSyrk && !t2_map_term(&q.tt, p.t[0], three_d)) return cudaErrorInvalidValue;
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
      ptiles[i] = p.kind == kSyrk ? q.tn * (q.tn + 1) / 2 : q.tn * q.tk;
      pkinds[i] = p.kind;
      total += ptiles[i];
    }
    a.count = n;
    a.total_tiles = (int)total;
    if (total == 0) continue;
#ifdef TC2_MAXCL
    const int clusters = periodic_workers(ptiles, pkinds, n, total, TC2_MAXCL);
#else
    const int clusters = periodic_workers(ptiles, pkinds, n, total, sms / 2);
#endif
    if (g_ring_set) {
      // the operands are raw fp32: without the ring they would be truncated -- fail loudly
      if (!three_d || !t2_ring_setup(a, prods + base, n, ptiles, clusters, s)) return cudaErrorNotSupported;
    }
    cudaError_t e;
    if (a.ring) {
      // The L2 ring's static schedule has CTAs waiting on one another's
      // rounding items and slot releases, so every CTA of the grid must be
      // resident at once: a cooperative launch guarantees it (the launch waits
      // for the SMs, or fails with cudaErrorCooperativeLaunchTooLarge, instead
      // of leaving resident CTAs spinning on CTAs that never start).
      cudaLaunchConfig_t cfg;
      std::memset(&cfg, 0, sizeof(cfg));
      cfg.gridDim = dim3(clusters * 2, 1, 1);
      cfg.blockDim = dim3(THREADS, 1, 1);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute attrs[2];
      attrs[0].id = cudaLaunchAttributeCooperative;
      attrs[0].val.cooperative = 1;
      cfg.attrs = attrs;
      cfg.numAttrs = 1;
      // ATA_TF32_RING_PIN=1 (A/B): an L2 access-policy window over the two rings marks
      // their lines persisting (slots are re-read by every tile of the wave) and the
      // launch's other traffic streaming
      static const bool pin = std::getenv("ATA_TF32_RING_PIN") != nullptr;
      if (pin) {
        int dev = 0, max_persist = 0, max_window = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        const size_t ring_bytes = (size_t)2 * a.rg.nslot * PR * a.rg.ncols * sizeof(float);
        if (max_persist > 0 && max_window > 0) {
          cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)max_persist);
          const size_t win = std::min(ring_bytes, (size_t)max_window);
          attrs[1].id = cudaLaunchAttributeAccessPolicyWindow;
          attrs[1].val.accessPolicyWindow.base_ptr = a.rg.ring[0];
          attrs[1].val.accessPolicyWindow.num_bytes = win;
          attrs[1].val.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)max_persist / (double)win);
          attrs[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
          attrs[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
          cfg.numAttrs = 2;
          static bool said = false;
          if (!said) {
            said = true;
            std::fprintf(stderr, "[ata] TF32 ring pinned: ring %zu B, window %zu B, persisting L2 %d B\n", ring_bytes,
                         win, max_persist);
          }
        }
      }
      e = cudaLaunchKernelEx(&cfg, prod_tf32_2sm_kernel, a);
    } else {
      prod_tf32_2sm_kernel<<<clusters * 2, THREADS, smem, s>>>(a);
      e = cudaGetLastError();
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace ata
