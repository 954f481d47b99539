// FP64 generalized-product kernel: persistent, warp-specialised (sm_100a, DMMA.8x8x4).
//
// Product semantics (shared with gemm_f64.cu / gemm_f32.cu):
//     D_d[:r_d, :c_d] (+)= sign_d * alpha * (sum_i s_i S_i)^T (sum_j t_j T_j)
// - up to two zero-extended operand terms per side: the Strassen pre-additions
//   (strassen.py:195-203) fused into the tile load;
// - up to four truncated destinations: the Strassen post-additions
//   (strassen.py:238-275 through add_truncated, matrix.py:218-239) fused into the
//   epilogue;
// - kind kSyrk = naive_syrk_lower (matrix.py:292-311) on lower-triangle tiles,
//   diagonal tiles masked on store (strict upper never touched, ata.py:121-123).
//
// Structure (one CTA per SM, persistent):
//   warpgroup 0 (128 threads, 40 regs)  producer: fetches output tiles from a
//       global work counter in launch order, streams [BK x 128] operand windows
//       with cp.async (16 B, or 8 B for odd pitches; zero-fill outside each
//       term window) into a STAGES-deep smem ring, combines two-term operands
//       in place once its own copies land, publishes through "full" mbarriers.
//   warpgroups 1-2 (256 threads, 232 regs)  consumers: 2 x 4 warps, 64 x 32
//       accumulators of 8x8 DMMA blocks read straight from padded smem rows,
//       release stages through "empty" mbarriers.  Epilogue: signed, truncated
//       RMW of every destination; a destination shared by several products of
//       the launch (a C quadrant of one Strassen node) is accumulated in
//       product order through per-tile turn counters, so results are bitwise
//       deterministic and a whole Strassen node (or level) is ONE launch
//       (no wave-quantisation tail per product).
// Deadlock freedom: tiles are handed out in increasing order and a tile only
// waits for turns of strictly earlier tiles, which are already running.
#include <cstdio>
#include <cstdlib>

#include <unordered_map>
#include <map>
#include <mutex>
#include <vector>
#include <cstring>
#include <type_traits>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "ata_common.cuh"

namespace ata {

#ifndef WS_PRODUCER_SUM
#define WS_PRODUCER_SUM 0  // 1: the producers add two-term operands in place (the old path)
#endif
#ifndef WS_CW
#define WS_CW 8  // consumer warps: 8 (2 x 4 grid of 64 x 32 warp tiles) or 16 (4 x 4 of 32 x 32)
#endif
namespace ws64 {
constexpr int BM = 128, BN = 128, LD = BM + 4;
constexpr int CONSUMERS = WS_CW, PRODUCERS = 128, THREADS = CONSUMERS * 32 + PRODUCERS;
// setmaxnreg split of the launch allocation: 8 warps 128*40 + 256*232 = 384*168;
// 16 warps 128*40 + 512*104 <= 640*96
constexpr int PRODUCER_REGS = 40, CONSUMER_REGS = CONSUMERS == 8 ? 232 : 104;
constexpr int WTM = CONSUMERS == 8 ? 8 : 4, WTN = 4;  // 64 x 32 or 32 x 32 per consumer warp
constexpr int SMEM_BUDGET = 225 * 1024;
constexpr int TSLOTS = 3;        // tile-info ring capacity (device-memory descriptors use 3 slots, parameter-space 2)
}  // namespace ws64

__device__ __forceinline__ void dmma_ws(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cpasync(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// The producer warpgroup copies a BK x 128 window of term t (rows l0.., cols c0..).
template <int BK, bool VEC16>
__device__ __forceinline__ void ws_load(double* buf, const DTerm<double>& t, int l0, int c0, int pt) {
  using namespace ws64;
  if (VEC16) {
#pragma unroll
    for (int i = 0; i < BK * (BM / 2) / PRODUCERS; ++i) {
      const int id = pt + i * PRODUCERS;
      const int r = id >> 6;  // BM/2 = 64 chunks per row
      const int c = (id & 63) * 2;
      const int gl = l0 + r, gc = c0 + c;
      int bytes = 0;
      if (gl < t.rows) {
        const int left = t.cols - gc;
        bytes = left >= 2 ? 16 : (left == 1 ? 8 : 0);
      }
      const double* src = bytes ? t.p + (long long)gl * t.ld + gc : t.p;
      cp_async_16(buf + r * LD + c, src, bytes);
    }
  } else {
#pragma unroll
    for (int i = 0; i < BK * BM / PRODUCERS; ++i) {
      const int id = pt + i * PRODUCERS;
      const int r = id >> 7;
      const int c = id & 127;
      const int gl = l0 + r, gc = c0 + c;
      const int bytes = (gl < t.rows && gc < t.cols) ? 8 : 0;
      const double* src = bytes ? t.p + (long long)gl * t.ld + gc : t.p;
      cp_async_8(buf + r * LD + c, src, bytes);
    }
  }
}

template <int BK, bool VEC16>
__device__ __forceinline__ void ws_combine(double* x, const double* y, double sign, int pt) {
  using namespace ws64;
  if (VEC16) {
#pragma unroll
    for (int i = 0; i < BK * (BM / 2) / PRODUCERS; ++i) {
      const int id = pt + i * PRODUCERS;
      const int r = id >> 6;
      const int c = (id & 63) * 2;
      double2* px = reinterpret_cast<double2*>(x + r * LD + c);
      const double2 vy = *reinterpret_cast<const double2*>(y + r * LD + c);
      double2 v = *px;
      v.x = fma(sign, vy.x, v.x);
      v.y = fma(sign, vy.y, v.y);
      *px = v;
    }
  } else {
#pragma unroll
    for (int i = 0; i < BK * BM / PRODUCERS; ++i) {
      const int id = pt + i * PRODUCERS;
      const int r = id >> 7;
      const int c = id & 127;
      x[r * LD + c] = fma(sign, y[r * LD + c], x[r * LD + c]);
    }
  }
}

__device__ __forceinline__ bool vec16_ok(const DTerm<double>& t) {
  return ((reinterpret_cast<uintptr_t>(t.p) & 15) == 0) && ((t.ld & 1) == 0);
}

struct TileInfo {
  int pi, ti, tj;
};

// product descriptors: in the kernel parameters (BatchArgsT) or in device memory (BatchArgsG)
template <typename T, int D, int B>
__device__ __forceinline__ const DProdT<T, D>& prod_of(const BatchArgsT<T, D, B>& a, int i) {
  return a.p[i];
}
template <typename T, int D>
__device__ __forceinline__ const DProdT<T, D>& prod_of(const BatchArgsG<T, D>& a, int i) {
  return a.gp[i];
}
template <typename T, int D, int B>
__device__ __forceinline__ int prod_index(const BatchArgsT<T, D, B>& a, int tile) {
  int pi = 0;
  while (pi + 1 < a.count && tile >= a.p[pi + 1].tile_begin) ++pi;
  return pi;
}
template <typename T, int D>
__device__ __forceinline__ int prod_index(const BatchArgsG<T, D>& a, int tile) {
  return __ldg(a.tile_prod + tile);
}

// How a role holds its tile's descriptor: parameter-space descriptors by
// reference (constant bank), device-memory descriptors by value (registers /
// local memory) -- global loads could not be hoisted across the epilogue's
// stores and would be re-issued per element.
template <typename Args>
struct ProdHold {
  using type = const DProdT<double, kMaxDests>&;
};
template <int B>
struct ProdHold<BatchArgsT<double, kNarrowDests, B>> {
  using type = const DProdT<double, kNarrowDests>&;
};
template <>
struct ProdHold<BatchArgsGlobal64> {
  using type = const DProdT<double, kNarrowDests>;
};

template <typename Args>
__device__ __forceinline__ TileInfo decode_tile(const Args& args, int tile) {
  const int pi = prod_index(args, tile);
  const auto& P = prod_of(args, pi);
  const int local = tile - P.tile_begin;
  TileInfo t;
  t.pi = pi;
  if (P.kind == kSyrk) {
    int r = (int)((sqrt(8.0 * (double)local + 1.0) - 1.0) * 0.5);
    while ((r + 1) * (r + 2) / 2 <= local) ++r;
    while (r * (r + 1) / 2 > local) --r;
    t.ti = r;
    t.tj = local - r * (r + 1) / 2;
  } else {
    // grouped raster: 8 tile-rows per group, column-major inside the group
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

// Epilogue of one output tile (shared by the cp.async- and TMA-fed kernels):
// signed, truncated writes of every destination; a destination region shared
// by several products of the launch is accumulated in product order through
// per-tile turn counters.
template <typename Args, typename PD>
__device__ __forceinline__ void ws_epilogue(const Args& args, const PD& P, const TileInfo& tl,
                                            const double (&acc)[ws64::WTM][ws64::WTN][2], int wm, int wn,
                                            int g, int q, int ctid) {
  using namespace ws64;
  const bool syrk = P.kind == kSyrk;
  const int i0 = tl.ti * BM, j0 = tl.tj * BN;
  const int nd = P.nd;
  const bool accumulate = P.accumulate != 0;
  for (int d = 0; d < ((args.dbg & 2) ? 0 : nd); ++d) {
    const DDest<double>& D = P.d[d];
    const double scale = args.alpha * D.sign;
    if (i0 >= D.rows || j0 >= D.cols) continue;  // tile entirely outside this window
    int* sem = nullptr;
    int turn = 0;
    if (D.sem >= 0 && !(args.dbg & 1)) {
      // turn = earlier products of the launch whose window in this region covers the tile
      for (int q = 0; q < tl.pi; ++q)
        for (int e = 0; e < prod_of(args, q).nd; ++e) {
          const DDest<double>& E = prod_of(args, q).d[e];
          if (E.sem == D.sem && i0 < E.rows && j0 < E.cols) ++turn;
        }
      sem = args.sync + D.sem + tl.ti * D.sem_ld + tl.tj;
      if (ctid == 0) {
        // bounded wait: a broken ordering invariant traps (launch error) instead of hanging
        uint64_t t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while (ld_acquire(sem) != turn) {
          __nanosleep(64);
          uint64_t t1;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
          if (t1 - t0 > 20000000000ull) __trap();
        }
      }
      named_sync(2, CONSUMERS * 32);
    }
#pragma unroll
    for (int r = 0; r < WTM; ++r) {
      const int row = i0 + wm * (WTM * 8) + r * 8 + g;
      if (row >= D.rows) continue;
      double* drow = D.p + (long long)row * D.ld;
#pragma unroll
      for (int c = 0; c < WTN; ++c) {
        const int col = j0 + wn * (WTN * 8) + c * 8 + q * 2;
        if (col + 1 < D.cols && (!syrk || col + 1 <= row) &&
            ((reinterpret_cast<uintptr_t>(drow + col) & 15) == 0)) {
          double2* p2 = reinterpret_cast<double2*>(drow + col);
          double2 v = make_double2(scale * acc[r][c][0], scale * acc[r][c][1]);
          if (accumulate) {
            const double2 o = __ldcg(p2);  // L2: another SM may have written it this launch
            v.x += o.x;
            v.y += o.y;
          }
          __stcg(p2, v);
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cc = col + e;
            if (cc < D.cols && (!syrk || cc <= row)) {
              const double v = scale * acc[r][c][e];
              __stcg(drow + cc, accumulate ? __ldcg(drow + cc) + v : v);
            }
          }
        }
      }
    }
    if (sem != nullptr) {
      __threadfence();
      named_sync(2, CONSUMERS * 32);
      if (ctid == 0) st_release(sem, turn + 1);
    }
  }
}

template <int BK, int NS, int NT, int STAGES, typename Args>
__global__ void __launch_bounds__(ws64::THREADS, 1)
    prod_f64_ws_kernel(const __grid_constant__ Args args) {
  using namespace ws64;
  constexpr int BUF = BK * LD;  // doubles per operand buffer
  constexpr int STAGE = (NS + NT) * BUF;
  extern __shared__ __align__(128) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + TSLOTS;
  int* tinfo = reinterpret_cast<int*>(tempty + TSLOTS);  // TSLOTS entries
  int* bcast = tinfo + TSLOTS;                            // producer-internal broadcast

  // Device-memory descriptors (BatchArgsGlobal64, thousands of small products):
  // the producers copy each tile's descriptor into a shared slot and decode
  // the tile once; consumers read both from the slot and release it after
  // their epilogue.  Parameter-space descriptors need none of it.
  constexpr bool kSmemDesc = std::is_same<Args, BatchArgsGlobal64>::value;
  constexpr int kSlots = kSmemDesc ? 3 : 2;
  __shared__ __align__(16) unsigned char
      pdesc_raw[kSmemDesc ? kSlots * sizeof(DProdT<double, kNarrowDests>) : 16];
  __shared__ int tdec[kSmemDesc ? kSlots : 1][3];  // decoded tile (product, tile row, tile col) per slot
  const int tid = threadIdx.x;
  const int warp = tid >> 5;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], PRODUCERS);
      mbar_init(&empty[s], CONSUMERS);
    }
    for (int s = 0; s < TSLOTS; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (tid < PRODUCERS) {
    // ===================== producer warpgroup =====================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PRODUCER_REGS));
    const int pt = tid;
    int kstep = 0;  // global k-step counter (stage ring position)
    for (int it = 0;; ++it) {
      if (pt == 0) *bcast = args.dynamic ? atomicAdd(args.sync, 1) : (int)(blockIdx.x + it * gridDim.x);
      named_sync(1, PRODUCERS);
      const int tile = *bcast;
      named_sync(1, PRODUCERS);
      const int slot = it % kSlots;
      using PD = std::remove_cv_t<std::remove_reference_t<decltype(prod_of(args, 0))>>;
      const PD* Pp;
      TileInfo tl;
      if constexpr (kSmemDesc) {
        // the slot (tile index, decoded tile, descriptor copy) is free once the
        // consumers have finished the tile that last used it
        if (pt == 0 && it >= kSlots) mbar_wait(&tempty[slot], ((it / kSlots) - 1) & 1);
        named_sync(1, PRODUCERS);
        if (tile >= args.total_tiles) {
          if (pt == 0) {
            tinfo[slot] = tile;
            mbar_arrive(&tfull[slot]);
          }
          break;
        }
        tl = decode_tile(args, tile);
        // the producers (40 registers) read the copy too (a by-value copy would live in local memory)
        const uint32_t* src = reinterpret_cast<const uint32_t*>(args.gp + tl.pi);
        uint32_t* dst = reinterpret_cast<uint32_t*>(pdesc_raw) + slot * (sizeof(PD) / 4);
        for (int i = pt; i < (int)(sizeof(PD) / 4); i += PRODUCERS) dst[i] = __ldg(src + i);
        Pp = reinterpret_cast<const PD*>(dst);
        named_sync(1, PRODUCERS);
        if (pt == 0) {
          tinfo[slot] = tile;
          tdec[slot][0] = tl.pi;
          tdec[slot][1] = tl.ti;
          tdec[slot][2] = tl.tj;
          mbar_arrive(&tfull[slot]);   // release: the descriptor copy and decoded tile
        }
      } else {
        if (pt == 0) {
          if (it >= kSlots) mbar_wait(&tempty[slot], ((it / kSlots) - 1) & 1);
          tinfo[slot] = tile;
          mbar_arrive(&tfull[slot]);
        }
        if (tile >= args.total_tiles) break;
        tl = decode_tile(args, tile);
        Pp = &prod_of(args, tl.pi);
      }
      const PD& P = *Pp;
      const bool syrk = P.kind == kSyrk;
      const bool same = syrk && tl.ti == tl.tj;
      const int ns = P.ns, nt = syrk ? 1 : P.nt;
      const int i0 = tl.ti * BM, j0 = tl.tj * BN;
      const DTerm<double>& S0 = P.s[0];
      const DTerm<double>& S1 = P.s[1];
      const DTerm<double>& T0 = syrk ? P.s[0] : P.t[0];
      const DTerm<double>& T1 = P.t[1];
      const bool vs = vec16_ok(S0) && (ns < 2 || vec16_ok(S1));
      const bool vt = vec16_ok(T0) && (nt < 2 || vec16_ok(T1));
      // two-term operands: both terms land in their own buffers and the
      // consumers add them while loading fragments (WS_PRODUCER_SUM: the
      // producers combine in place instead -- measured slower: the in-place
      // pass throttles the producer ring)
      const bool comb = WS_PRODUCER_SUM && ((NS == 2 && ns == 2) || (NT == 2 && nt == 2));
      const int KT = (P.m + BK - 1) / BK;
      auto issue = [&](int kt, int ring) {
        double* base = smem + (ring % STAGES) * STAGE;
        const int l0 = kt * BK;
        if (vs) ws_load<BK, true>(base, S0, l0, i0, pt);
        else ws_load<BK, false>(base, S0, l0, i0, pt);
        if (NS == 2 && ns == 2) {
          if (vs) ws_load<BK, true>(base + BUF, S1, l0, i0, pt);
          else ws_load<BK, false>(base + BUF, S1, l0, i0, pt);
        }
        if (!same) {
          double* tb = base + NS * BUF;
          if (vt) ws_load<BK, true>(tb, T0, l0, j0, pt);
          else ws_load<BK, false>(tb, T0, l0, j0, pt);
          if (NT == 2 && nt == 2) {
            if (vt) ws_load<BK, true>(tb + BUF, T1, l0, j0, pt);
            else ws_load<BK, false>(tb + BUF, T1, l0, j0, pt);
          }
        }
      };
      auto finish = [&](int ring) {  // combine two-term operands of a stage, publish it
        double* base = smem + (ring % STAGES) * STAGE;
        if (NS == 2 && ns == 2) {
          if (vs) ws_combine<BK, true>(base, base + BUF, S1.sign, pt);
          else ws_combine<BK, false>(base, base + BUF, S1.sign, pt);
        }
        if (NT == 2 && nt == 2) {
          double* tb = base + NS * BUF;
          if (vt) ws_combine<BK, true>(tb, tb + BUF, T1.sign, pt);
          else ws_combine<BK, false>(tb, tb + BUF, T1.sign, pt);
        }
        mbar_arrive(&full[ring % STAGES]);
      };
      // two-term operands: stage kt is combined once its copies have landed,
      // LAG stages behind the newest issue (LAG groups stay in flight)
      constexpr int LAG = STAGES > 3 ? STAGES - 2 : 1;
      for (int kt = 0; kt < KT; ++kt, ++kstep) {
        const int s = kstep % STAGES;
        if (kstep >= STAGES) mbar_wait(&empty[s], ((kstep / STAGES) - 1) & 1);
#ifdef WS_AB_NOLOAD   // A/B probe: no operand traffic (stages publish stale data)
        mbar_arrive(&full[s]);
        continue;
#endif
        issue(kt, kstep);
        if (!comb) {
          mbar_arrive_cpasync(&full[s]);
        } else {
          cp_async_commit();
          if (kt >= LAG) {
            cp_async_wait<LAG>();
            finish(kstep - LAG);
          }
        }
      }
      if (comb) {
        cp_async_wait<0>();
        for (int d = (KT < LAG ? KT : LAG); d >= 1; --d) finish(kstep - d);
      }
    }
    cp_async_wait<0>();
    return;
  }

  // ===================== consumer warpgroups =====================
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CONSUMER_REGS));
  const int ctid = tid - PRODUCERS;
  const int lane = tid & 31;
  const int cw = warp - PRODUCERS / 32;
  const int wm = cw >> 2, wn = cw & 3;  // 2 x 4 consumer warps
  const int g = lane >> 2, q = lane & 3;
  int kstep = 0;
  for (int it = 0;; ++it) {
    const int slot = it % kSlots;
    mbar_wait(&tfull[slot], (it / kSlots) & 1);
    const int tile = tinfo[slot];
    TileInfo tl;
    if constexpr (kSmemDesc) {
      if (tile >= args.total_tiles) break;
      tl.pi = tdec[slot][0];
      tl.ti = tdec[slot][1];
      tl.tj = tdec[slot][2];
    } else {   // parameter-space descriptor: the slot is free at once
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[slot]);
      if (tile >= args.total_tiles) break;
      tl = decode_tile(args, tile);
    }
    using PDc = std::remove_cv_t<std::remove_reference_t<decltype(prod_of(args, 0))>>;
    const PDc& P = kSmemDesc ? *reinterpret_cast<const PDc*>(pdesc_raw + slot * sizeof(PDc))
                             : prod_of(args, tl.pi);
    const bool syrk = P.kind == kSyrk;
    const bool same = syrk && tl.ti == tl.tj;
    const int KT = (P.m + BK - 1) / BK;

    double acc[WTM][WTN][2];
#pragma unroll
    for (int r = 0; r < WTM; ++r)
#pragma unroll
      for (int c = 0; c < WTN; ++c) acc[r][c][0] = acc[r][c][1] = 0.0;

    const int aoff = wm * (WTM * 8) + g + q * LD;
    const int boff = (same ? 0 : NS * BUF) + wn * (WTN * 8) + g + q * LD;
    // second operand terms (consumer-side sum): S1 / T1 sit one buffer after S0 / T0
    const bool two_a = !WS_PRODUCER_SUM && NS == 2 && P.ns == 2;
    const bool two_b = !WS_PRODUCER_SUM && (same ? two_a : (NT == 2 && P.nt == 2));
    const double sa = two_a ? P.s[1].sign : 0.0;
    const double sb = same ? sa : (two_b ? P.t[1].sign : 0.0);
    for (int kt = 0; kt < KT; ++kt, ++kstep) {
      const int s = kstep % STAGES;
#ifndef WS_AB_NOFULLWAIT   // A/B probe: consumers never wait for data
      mbar_wait(&full[s], (kstep / STAGES) & 1);
#endif
      const double* As = smem + s * STAGE + aoff;
      const double* Bs = smem + s * STAGE + boff;
#pragma unroll
      for (int kk = 0; kk < BK / 4; ++kk) {
        double a[WTM], b[WTN];
#pragma unroll
        for (int r = 0; r < WTM; ++r) a[r] = As[kk * 4 * LD + r * 8];
#pragma unroll
        for (int c = 0; c < WTN; ++c) b[c] = Bs[kk * 4 * LD + c * 8];
        if (NS == 2 && two_a) {
#pragma unroll
          for (int r = 0; r < WTM; ++r) a[r] = fma(sa, As[BUF + kk * 4 * LD + r * 8], a[r]);
        }
        if ((NS == 2 || NT == 2) && two_b) {
#pragma unroll
          for (int c = 0; c < WTN; ++c) b[c] = fma(sb, Bs[BUF + kk * 4 * LD + c * 8], b[c]);
        }
#pragma unroll
        for (int r = 0; r < WTM; ++r)
#pragma unroll
          for (int c = 0; c < WTN; ++c) dmma_ws(acc[r][c], a[r], b[c]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    // ---- epilogue: fused post-additions into up to four destinations ----
    ws_epilogue(args, P, tl, acc, wm, wn, g, q, ctid);
    if (kSmemDesc) {    // the shared descriptor copy was read up to here
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[slot]);
    }
  }
}


static int num_sms() { return ata::sm_count(); }

template <int BK, int NS, int NT, typename Args>
static cudaError_t ws_kernel_launch(const Args& a, long long total, cudaStream_t s) {
  using namespace ws64;
  constexpr int STAGE_BYTES = (NS + NT) * BK * LD * 8;
  constexpr int STAGES =
      (SMEM_BUDGET - 1024) / STAGE_BYTES > 8 ? 8 : (SMEM_BUDGET - 1024) / STAGE_BYTES;
  static_assert(STAGES >= 2, "smem");
  const size_t smem = (size_t)STAGES * STAGE_BYTES + (2 * STAGES + 2 * TSLOTS) * sizeof(uint64_t) +
                      (TSLOTS + 2) * sizeof(int);
  auto kern = prod_f64_ws_kernel<BK, NS, NT, STAGES, Args>;
  static std::atomic<unsigned long long> attr_set{0};
  if (cudaError_t e = ata::set_smem_attr(kern, smem, attr_set); e != cudaSuccess) return e;
  const int grid = (int)(total < num_sms() ? total : num_sms());
  kern<<<grid, THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

template <int BK, int NS, int NT, typename Args>
static cudaError_t launch_ws(Args a, cudaStream_t s) {
  using namespace ws64;
  long long total = 0;
  for (int i = 0; i < a.count; ++i) {
    auto& p = a.p[i];
    p.tn = (p.n + BM - 1) / BM;
    p.tk = (p.k + BN - 1) / BN;
    p.tile_begin = (int)total;
    total += p.kind == kSyrk ? (long long)p.tn * (p.tn + 1) / 2 : (long long)p.tn * p.tk;
  }
  if (total <= 0) return cudaSuccess;
  if (total > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  a.total_tiles = (int)total;
  // turn counters: regions were numbered by the executor (DDest.sem = region id + 1, 0 = none)
  int n_sync = 1;
  {
    int region_base[kMaxBatch * kMaxDests];
    int region_ld[kMaxBatch * kMaxDests];
    int region_rows[kMaxBatch * kMaxDests];
    int region_seen[kMaxBatch * kMaxDests];
    for (int r = 0; r < kMaxBatch * kMaxDests; ++r) region_base[r] = -1, region_ld[r] = 0, region_rows[r] = 0, region_seen[r] = 0;
    for (int i = 0; i < a.count; ++i)
      for (int d = 0; d < a.p[i].nd; ++d) {
        const int rg = a.p[i].d[d].sem;
        if (rg <= 0 || rg > kMaxBatch * kMaxDests) continue;
        region_ld[rg - 1] = max(region_ld[rg - 1], a.p[i].tk);
        region_rows[rg - 1] = max(region_rows[rg - 1], a.p[i].tn);
      }
    for (int r = 0; r < kMaxBatch * kMaxDests; ++r)
      if (region_ld[r] > 0) {
        region_base[r] = n_sync;
        n_sync += region_ld[r] * region_rows[r];
      }
    for (int i = 0; i < a.count; ++i)
      for (int d = 0; d < a.p[i].nd; ++d) {
        DDest<double>& D = a.p[i].d[d];
        const int rg = D.sem;
        if (rg <= 0 || rg > kMaxBatch * kMaxDests) {
          D.sem = -1;
          continue;
        }
        D.sem = region_base[rg - 1];
        D.sem_ld = region_ld[rg - 1];
        D.turn = region_seen[rg - 1]++;
      }
  }
  cudaError_t e = cudaSuccess;
  a.dynamic = n_sync > 1;
  { const char* e = std::getenv("ATA_DBG"); a.dbg = e ? std::atoi(e) : 0; }
  if (a.dynamic) {
    if (a.sync == nullptr || n_sync > a.n_sync) return cudaErrorInvalidValue;
    e = cudaMemsetAsync(a.sync, 0, (size_t)n_sync * sizeof(int), s);
    if (e != cudaSuccess) return e;
  }
  return ws_kernel_launch<BK, NS, NT>(a, total, s);
}

#ifndef WS2_BK
#define WS2_BK 16  // k-block rows of the two-term (fused Strassen sum) configurations
#endif

template <typename Args>
static cudaError_t launch_ws_any(const Args& a, cudaStream_t s) {
  int ns = 1, nt = 1;
  for (int i = 0; i < a.count; ++i) {
    ns = max(ns, a.p[i].ns);
    if (a.p[i].kind != kSyrk) nt = max(nt, a.p[i].nt);
  }
  static int bk = -1;
  if (bk < 0) {
    const char* e = std::getenv("ATA_WS_BK");
    // single-term leaves: 32-row k-blocks x 3 stages (c4 45.71 -> 45.97 TF/s, c3 40.43 ->
    // 40.54, c2 unchanged); ATA_WS_BK=16 selects 16-row k-blocks x 6 stages
    bk = e ? std::atoi(e) : 32;
  }
  if (bk == 32) {
    if (ns == 1 && nt == 1) return launch_ws<32, 1, 1>(a, s);
    if (ns == 2 && nt == 1) return launch_ws<16, 2, 1>(a, s);
    if (ns == 1 && nt == 2) return launch_ws<16, 1, 2>(a, s);
    return launch_ws<16, 2, 2>(a, s);
  }
  if (ns == 1 && nt == 1) return launch_ws<16, 1, 1>(a, s);
  if (ns == 2 && nt == 1) return launch_ws<WS2_BK, 2, 1>(a, s);
  if (ns == 1 && nt == 2) return launch_ws<WS2_BK, 1, 2>(a, s);
  return launch_ws<WS2_BK, 2, 2>(a, s);
}

cudaError_t launch_batch_f64_ws(const BatchArgs<double>& a, cudaStream_t s) { return launch_ws_any(a, s); }


// ===========================================================================
// TMA-fed variant (single-term operands).  Same warp roles, tiles, epilogue
// and tile queue as prod_f64_ws_kernel, but the operand windows reach shared
// memory through the tensor-memory accelerator: ONE producer thread issues,
// per k-block, one 3-D bulk tensor copy per operand ([8 panels][BK rows][16
// doubles], 128-byte swizzle) instead of 4096 16-byte cp.async per stage from
// 128 threads (measured: removing the cp.async traffic alone lifts the c4 leaf
// group from 33.3 to 35.2 TF/s, tools/f64_ab.py).  Rows / columns outside a
// window are zero-filled by the TMA unit (the reference's zero-extension).
//
// Bank-conflict-free fragment reads of the swizzled layout: a DMMA m8n8k4
// fragment lane (g, q) reads element (k = q, m/n = g); the k-slots of one DMMA
// are mapped to smem rows {x, x+2, x+4, x+6} (x = k-step parity) of an 8-row
// swizzle atom, whose 16-byte chunks the 128B swizzle spreads over all 32
// banks.  The contraction order inside a k-block is permuted accordingly (the
// same permutation for both operands).
// ===========================================================================
namespace wst {
#ifndef WST_BK
#define WST_BK 32     // k-block rows, single-term launches
#endif
#ifndef WST_BK2
#define WST_BK2 16    // k-block rows, launches with two-term (fused Strassen sum) operands
#endif
constexpr int PANELS = ws64::BM / 16;              // 16 doubles = one 128-byte swizzle row
// register split of the launch allocation (384 x 168 = 64512; setmaxnreg.inc can only
// draw what the CTA itself released): 128 producer threads x 72 (the spare warps run
// the riding operand sums, two rows = 8 loads in flight) + 256 consumer threads x 216
constexpr int PRODUCER_REGS = 72, CONSUMER_REGS = 216;
static_assert(PRODUCER_REGS * ws64::PRODUCERS + CONSUMER_REGS * ws64::CONSUMERS * 32 <= 168 * ws64::THREADS,
              "setmaxnreg split exceeds the launch allocation: the consumers' inc would block forever");
template <int BK>
constexpr int buf_bytes() { return BK * 128 * PANELS; }   // one operand term, one k-block
template <int BK, int NS, int NT>
constexpr int stage_bytes() { return (NS + NT) * buf_bytes<BK>(); }
template <int BK, int NS, int NT>
constexpr int stages() {
  return (ws64::SMEM_BUDGET - 2048) / stage_bytes<BK, NS, NT>() > 6 ? 6
                                                                  : (ws64::SMEM_BUDGET - 2048) / stage_bytes<BK, NS, NT>();
}
}  // namespace wst

// ---- riding operand sums ------------------------------------------------
// The Strassen pre-additions (strassen.py:195-203, one combo4 node = the five
// operand sums of one Strassen node's operand) of the NEXT leaf group are
// HBM-bound and independent of this launch's products, which are DMMA-bound and
// leave three of the four producer warps idle.  A launch may therefore carry a
// "ride": a list of combo4 nodes cut into chunks (64-column strips of kRideRows rows)
// that the spare warps claim from a global queue.  Nodes are ordered by phase;
// a node of phase p > 0 reads outputs of earlier phases and waits until every
// chunk of phase p - 1 is finished.  Chunks are claimed in increasing order and
// a chunk only ever waits for lower-numbered chunks (already claimed by running
// warps that never wait on later ones), so the wait is deadlock-free without
// any co-residency assumption.
struct RideNode {
  const double* src[4];
  double* dst[5];
  int srows[4], scols[4];   // source extents (zero beyond them)
  int sld, dld;             // the sources' common pitch, the outputs' common pitch
  int nsrc, ndst, rows, cp; // iteration extent: rows x cp column pairs (= every output's extent)
  unsigned long long codes; // output j: 8 bits at 8 j, base-4 digits over the sources (1: +, 2: -)
  int strips;               // ceil(cp / 32): a chunk is one 64-column strip of kRideRows rows
  int chunk_begin;          // first chunk of this node in the ride's chunk space
  int phase;
  int wait_chunks;          // chunks of phase - 1 that must be finished first (0: none)
};
static_assert(sizeof(RideNode) % 8 == 0, "RideNode is copied as 32-bit words and stored in 8-byte blobs");
constexpr int kRideRows = 64;   // rows per chunk: 64 rows x 32 column pairs (16 bytes per lane and row)

struct TmaBatch64 {
  int count;
  int total_tiles;
  double alpha;
  int* sync;
  int n_sync;
  int dynamic;
  int dbg;
  int map3d;                                    // 1: 3-D maps (one box per operand); 0: 2-D maps, 8 boxes
  const CUtensorMap* maps;                      // device array [4 * count]: S0, S1, T0, T1 of each product
  const DProdT<double, kNarrowDests>* gp;       // device array [count]
  const int* tile_prod;                         // device array [total_tiles]
  int ride_nodes, ride_chunks;                  // riding operand sums (0: none)
  const RideNode* ride;                         // device array [ride_nodes]
  int* ride_sync;                               // [0] chunk queue, [1 + p] finished chunks of phase p
};

// A/B probes (tools/ride_ab.py): RIDE_AB_NOLOAD / NOSTORE / NOADD drop one ingredient of
// the riding sums (wrong results, timing only)
__device__ __forceinline__ double2 ride_ld(const double* p) {
  double2 v;
#ifdef RIDE_AB_NOLOAD
  return make_double2((double)(reinterpret_cast<uintptr_t>(p) & 255), 1.0);
#endif
  asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void ride_st(double* p, double2 v) {
#ifdef RIDE_AB_NOSTORE
  if (v.x != 1.2345e300) return;
#endif
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// base-4 coefficient digits (digit q of output j at bit 8 j + 2 q: 1 = +, 2 = -) of the
// five operand sums of strassen.py:234-273 over the quadrants (X11, X12, X21, X22):
//   S side: X11+X22, X12+X22, X11+X21, X12-X11, X21-X22
//   T side: X11+X22, X12-X22, X21-X11, X11+X12, X21+X22
constexpr unsigned long long ride_codes(int o0, int o1, int o2, int o3, int o4) {
  return (unsigned long long)o0 | (unsigned long long)o1 << 8 | (unsigned long long)o2 << 16 |
         (unsigned long long)o3 << 24 | (unsigned long long)o4 << 32;
}
constexpr unsigned long long kRideCodesS = ride_codes(1 | 1 << 6, 1 << 2 | 1 << 6, 1 | 1 << 4, 2 | 1 << 2, 1 << 4 | 2 << 6);
constexpr unsigned long long kRideCodesT = ride_codes(1 | 1 << 6, 1 << 2 | 2 << 6, 2 | 1 << 4, 1 | 1 << 2, 1 << 4 | 1 << 6);

// nr rows of one strip: per row, 4 independent 16-byte loads, the signed sums, 5 stores.
// CODES != 0: compile-time coefficients (all five outputs present); 0: decode `codes`.
// A two-term sum (every operand sum of a Strassen node) is a plain store of its + term
// followed by an L2 reduction of the other (red.global.add.f64 -- SASS REDG.E.ADD.F64.RN --
// the - sign applied with an integer XOR): the same IEEE round-to-nearest sum, computed by
// the L2 atomic units, so no instruction of the ride enters the FP64 pipe the DMMAs own
// (a DADD queued ~300 cycles behind the consumers' DMMA bursts).  A thread's store and
// reduction to one address are ordered (same-address program order).  -DRIDE_DADD: the
// sums in registers (the first version; measured c4 1380 vs 1367 ms); -DRIDE_RED_MASK=bits:
// only those outputs go through L2 reductions, the others are added in registers.
__device__ __forceinline__ double ride_flip(double x) {
  // (asm: written as C++ the XOR is folded into an fneg, which ptxas emits as a DADD)
  unsigned lo, hi;
  double y;
  asm volatile("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(x));
  asm volatile("xor.b32 %0, %0, 0x80000000;" : "+r"(hi));
  asm volatile("mov.b64 %0, {%1, %2};" : "=d"(y) : "r"(lo), "r"(hi));
  return y;
}
// (RIDE_POLICY: stores and reductions carry an L2 evict_first policy, so the sums stream
// through L2 without displacing the operand panels the products re-read; RIDE_ST_CS: the
// store alone is a streaming store)
__device__ __forceinline__ unsigned long long ride_policy() {
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void ride_red(double* p, double2 v) {
#ifdef RIDE_AB_NORED
  if (v.x != 1.2345e300) return;
#endif
#ifdef RIDE_POLICY
  const unsigned long long pol = ride_policy();
  asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v.x), "l"(pol) : "memory");
  asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p + 1), "d"(v.y), "l"(pol) : "memory");
#else
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v.x) : "memory");
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p + 1), "d"(v.y) : "memory");
#endif
}
__device__ __forceinline__ void ride_st_keep(double* p, double2 v) {
#ifdef RIDE_AB_NOSTORE
  if (v.x != 1.2345e300) return;
#endif
#if defined(RIDE_POLICY)
  const unsigned long long pol = ride_policy();
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
#elif defined(RIDE_ST_CS)
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
#else
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
#endif
}
constexpr int ride_plus_term(unsigned code) {
  return (code & 3u) == 1 ? 0 : ((code >> 2) & 3u) == 1 ? 1 : ((code >> 4) & 3u) == 1 ? 2 : 3;
}
constexpr int ride_other_term(unsigned code) {
  const int a = ride_plus_term(code);
  return (a != 0 && (code & 3u)) ? 0 : (a != 1 && ((code >> 2) & 3u)) ? 1 : (a != 2 && ((code >> 4) & 3u)) ? 2 : 3;
}

template <unsigned long long CODES>
__device__ __forceinline__ void ride_out(const double2 (&v)[4], double* (&dp)[5], long long dld,
                                         unsigned long long codes) {
#ifndef RIDE_RED_MASK
#ifdef RIDE_DADD
#define RIDE_RED_MASK 0
#else
#define RIDE_RED_MASK 31   // bit j: output j of a compile-time pattern is a store + L2 reduction
#endif
#endif
  if (CODES != 0) {
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const unsigned code = (unsigned)(CODES >> (8 * j)) & 255u;
      if (RIDE_RED_MASK >> j & 1) ride_st_keep(dp[j], v[ride_plus_term(code)]);
    }
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      if (!(RIDE_RED_MASK >> j & 1)) continue;
      const unsigned code = (unsigned)(CODES >> (8 * j)) & 255u;
      const int qb = ride_other_term(code);
      double2 t = v[qb];
      if (((code >> (2 * qb)) & 3u) == 2) t = make_double2(ride_flip(t.x), ride_flip(t.y));
      ride_red(dp[j], t);
      dp[j] += dld;
    }
  }
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    if (CODES == 0 && dp[j] == nullptr) continue;
    if (CODES != 0 && (RIDE_RED_MASK >> j & 1)) continue;
    const unsigned code = (unsigned)((CODES ? CODES : codes) >> (8 * j)) & 255u;
    double2 o = make_double2(0.0, 0.0);
    bool first = true;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const unsigned cq = (code >> (2 * q)) & 3u;
      if (CODES != 0 && first && cq == 1) {   // leading +1 term: no add (0.0 + x == x)
        o = v[q];
      }
#ifndef RIDE_AB_NOADD
      else if (cq == 1) {
        o.x += v[q].x, o.y += v[q].y;
      } else if (cq == 2) {
        o.x -= v[q].x, o.y -= v[q].y;
      }
#endif
      if (cq != 0) first = false;
    }
    ride_st(dp[j], o);
    dp[j] += dld;
  }
}
// FULL: every source covers all rows of the chunk (no per-row limit tests)
template <bool FULL>
__device__ __forceinline__ void ride_in(double2 (&v)[4], const double* (&sp)[4], const int (&lim)[4], int i,
                                        long long sld) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (FULL) {
      v[q] = ride_ld(sp[q]);
    } else {
      v[q] = make_double2(0.0, 0.0);
      if (i < lim[q]) v[q] = ride_ld(sp[q]);
    }
    sp[q] += sld;
  }
}
template <unsigned long long CODES, bool FULL>
__device__ __forceinline__ void ride_rows(const double* (&sp)[4], const int (&lim)[4], double* (&dp)[5],
                                          long long sld, long long dld, int nr, unsigned long long codes) {
  int i = 0;
#ifdef RIDE_PIPE
  if (CODES != 0 && nr >= 2) {   // rows alternate between two register sets: the next row's loads
    double2 v[4], w[4];          // are issued before the current row's stores
    ride_in<FULL>(v, sp, lim, 0, sld);
    for (; i + 1 < nr; i += 2) {
      ride_in<FULL>(w, sp, lim, i + 1, sld);
      ride_out<CODES>(v, dp, dld, codes);
      if (i + 2 < nr) ride_in<FULL>(v, sp, lim, i + 2, sld);
      ride_out<CODES>(w, dp, dld, codes);
    }
    if (i < nr) ride_out<CODES>(v, dp, dld, codes);
    return;
  }
#endif
  if (CODES != 0) {   // two rows per trip: 8 independent 16-byte loads in flight per lane
    for (; i + 1 < nr; i += 2) {
      double2 v[4], w[4];
      ride_in<FULL>(v, sp, lim, i, sld);
      ride_in<FULL>(w, sp, lim, i + 1, sld);
      ride_out<CODES>(v, dp, dld, codes);
      ride_out<CODES>(w, dp, dld, codes);
    }
  }
  for (; i < nr; ++i) {
    double2 v[4];
    ride_in<FULL>(v, sp, lim, i, sld);
    ride_out<CODES>(v, dp, dld, codes);
  }
}

// A spare producer warp: claim chunks until the queue is empty.  `node` is the
// warp's private shared-memory copy of the node it is working on.  A chunk is a
// strip of 32 column pairs (one per lane) x kRideRows rows; everything the inner
// loop needs lives in registers (pointers advance by the common pitches), so its
// loads issue back to back: 4 x 16 bytes in flight per lane.
__device__ __forceinline__ void ride_worker(const TmaBatch64& args, RideNode* node, int lane) {
  int cur = -1;
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(args.ride_sync, 1);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= args.ride_chunks) break;
    int ni = cur < 0 ? 0 : cur;
    while (ni + 1 < args.ride_nodes && c >= __ldg(&args.ride[ni + 1].chunk_begin)) ++ni;
    if (ni != cur) {
      __syncwarp();
      const uint32_t* src = reinterpret_cast<const uint32_t*>(args.ride + ni);
      uint32_t* dst = reinterpret_cast<uint32_t*>(node);
      for (int i = lane; i < (int)(sizeof(RideNode) / 4); i += 32) dst[i] = __ldg(src + i);
      __syncwarp();
      cur = ni;
      if (node->wait_chunks > 0) {
        if (lane == 0) {
          const int* done = args.ride_sync + node->phase;   // = ride_sync + 1 + (phase - 1)
          uint64_t t0;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
          while (ld_acquire(done) < node->wait_chunks) {
            __nanosleep(256);
            uint64_t t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            if (t1 - t0 > 20000000000ull) __trap();   // broken ordering invariant: fail the launch
          }
        }
        __syncwarp();
      }
    }
    const int local = c - node->chunk_begin;
    const int rb = local / node->strips, st = local - rb * node->strips;
    const int r0 = rb * kRideRows;
    const int nr = min(kRideRows, node->rows - r0);
    const int pc = st * 32 + lane;
    const int phase = node->phase;
    if (pc < node->cp) {
      const int col = 2 * pc;
      const long long sld = node->sld, dld = node->dld;
      const unsigned long long codes = node->codes;
      const double* sp[4];
      int lim[4];        // rows of this chunk inside source q (<= 0: none; the column test folds in)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool on = q < node->nsrc && col < node->scols[q];
        sp[q] = on ? node->src[q] + (long long)r0 * sld + col : nullptr;
        lim[q] = on ? node->srows[q] - r0 : 0;
      }
      double* dp[5];
#pragma unroll
      for (int j = 0; j < 5; ++j) dp[j] = j < node->ndst ? node->dst[j] + (long long)r0 * dld + col : nullptr;
      // the two coefficient patterns of a Strassen node's operand sums (auto_plan._S / _T)
      // run with compile-time coefficients; anything else decodes its digits per row
      const bool full = lim[0] >= nr && lim[1] >= nr && lim[2] >= nr && lim[3] >= nr;
      if (codes == kRideCodesS && node->ndst == 5) {
        if (full) ride_rows<kRideCodesS, true>(sp, lim, dp, sld, dld, nr, codes);
        else ride_rows<kRideCodesS, false>(sp, lim, dp, sld, dld, nr, codes);
      } else if (codes == kRideCodesT && node->ndst == 5) {
        if (full) ride_rows<kRideCodesT, true>(sp, lim, dp, sld, dld, nr, codes);
        else ride_rows<kRideCodesT, false>(sp, lim, dp, sld, dld, nr, codes);
      } else {
        ride_rows<0ull, false>(sp, lim, dp, sld, dld, nr, codes);
      }
    }
    // publish the chunk: every lane's stores, then one count
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicAdd(args.ride_sync + 1 + phase, 1);
  }
}

__device__ __forceinline__ const DProdT<double, kNarrowDests>& prod_of(const TmaBatch64& a, int i) {
  return a.gp[i];
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// one operand term's k-block: a 3-D box, or eight 2-D boxes of [BK rows][16 doubles]
// (2-D maps start 0 or 1 element before the window: col0 = its 8-byte misalignment)
template <int BK>
__device__ __forceinline__ void tma_term(uint32_t dst, const CUtensorMap* map, const DTerm<double>& t, bool map3d,
                                         int kt, int c0, uint32_t bar) {
  if (map3d) {
    tma_load_3d(dst, map, 0, kt * BK, c0 / 16, bar);
  } else {
    const int col0 = (int)((reinterpret_cast<uintptr_t>(t.p) >> 3) & 1);
#pragma unroll
    for (int p = 0; p < wst::PANELS; ++p) tma_load_2d(dst + p * BK * 128, map, col0 + c0 + 16 * p, kt * BK, bar);
  }
}
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

// NS / NT: operand terms per side (2: a Strassen operand sum X + s Y read as two
// zero-extended windows and added as the fragments are loaded -- the pre-addition
// fused into the product, no operand-sum buffer in HBM).  Products with fewer
// terms than the launch's NS / NT run in the same launch.
template <int BK, int NS, int NT>
__global__ void __launch_bounds__(ws64::THREADS, 1) prod_f64_tma_kernel(const __grid_constant__ TmaBatch64 args) {
  using namespace ws64;
  constexpr int BUF_BYTES = wst::buf_bytes<BK>();
  constexpr int STAGE_BYTES = wst::stage_bytes<BK, NS, NT>();
  constexpr int STAGES = wst::stages<BK, NS, NT>();
  static_assert(BK % 8 == 0 && STAGES >= 2, "TMA k-block");
  using PD = DProdT<double, kNarrowDests>;
  constexpr int kSlots = 3;
  extern __shared__ uint8_t tma_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tma_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + kSlots;
  int* tinfo = reinterpret_cast<int*>(tempty + kSlots);
  __shared__ __align__(16) unsigned char pdesc_raw[kSlots * sizeof(PD)];
  __shared__ int tdec[kSlots][3];
  __shared__ __align__(16) RideNode ride_node[3];   // one per spare producer warp
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMERS);
    }
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (tid < PRODUCERS) {
    // ===================== producer: one warp, one issuing thread =====================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(wst::PRODUCER_REGS));
    if (warp != 0) {
      // spare producer warps: the riding operand sums of the next leaf group
      if (args.ride_chunks > 0) ride_worker(args, &ride_node[warp - 1], lane);
      return;
    }
    int kstep = 0;
    for (int it = 0;; ++it) {
      int tile = 0;
      if (lane == 0) tile = args.dynamic ? atomicAdd(args.sync, 1) : (int)(blockIdx.x + it * gridDim.x);
      tile = __shfl_sync(0xffffffffu, tile, 0);
      const int slot = it % kSlots;
      if (lane == 0 && it >= kSlots) mbar_wait(&tempty[slot], ((it / kSlots) - 1) & 1);
      __syncwarp();
      if (tile >= args.total_tiles) {
        if (lane == 0) {
          tinfo[slot] = tile;
          mbar_arrive(&tfull[slot]);
        }
        break;
      }
      const int pi = __ldg(args.tile_prod + tile);
      const uint32_t* src = reinterpret_cast<const uint32_t*>(args.gp + pi);
      uint32_t* dst = reinterpret_cast<uint32_t*>(pdesc_raw) + slot * (sizeof(PD) / 4);
      for (int i = lane; i < (int)(sizeof(PD) / 4); i += 32) dst[i] = __ldg(src + i);
      __syncwarp();
      const PD& P = *reinterpret_cast<const PD*>(dst);
      const int local = tile - P.tile_begin;
      int ti, tj;
      if (P.kind == kSyrk) {
        int r = (int)((sqrt(8.0 * (double)local + 1.0) - 1.0) * 0.5);
        while ((r + 1) * (r + 2) / 2 <= local) ++r;
        while (r * (r + 1) / 2 > local) --r;
        ti = r;
        tj = local - r * (r + 1) / 2;
      } else {
        const int per_group = 8 * P.tk;
        const int grp = local / per_group;
        const int first = grp * 8;
        const int gsz = min(P.tn - first, 8);
        const int in = local - grp * per_group;
        ti = first + in % gsz;
        tj = in / gsz;
      }
      const bool same = P.kind == kSyrk && ti == tj;
      const int KT = (P.m + BK - 1) / BK;
      if (lane == 0) {
        tinfo[slot] = tile;
        tdec[slot][0] = pi;
        tdec[slot][1] = ti;
        tdec[slot][2] = tj;
        mbar_arrive(&tfull[slot]);   // release: descriptor copy and decoded tile
        // maps of product pi: [S0, S1, T0, T1] (4 per product)
        const CUtensorMap* ms = args.maps + 4 * pi;
        const CUtensorMap* mt = P.kind == kSyrk ? ms : ms + 2;
        const int ns = NS == 2 ? P.ns : 1, nt = P.kind == kSyrk ? ns : (NT == 2 ? P.nt : 1);
        const uint32_t bytes = (same ? ns : ns + nt) * BUF_BYTES;
        for (int kt = 0; kt < KT; ++kt, ++kstep) {
          const int s = kstep % STAGES;
          if (kstep >= STAGES) mbar_wait(&empty[s], ((kstep / STAGES) - 1) & 1);
          const uint32_t bar = smem_u32(&full[s]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                       : "memory");
          const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
          const bool m3 = args.map3d != 0;
          const DTerm<double>* tt = P.kind == kSyrk ? P.s : P.t;
          tma_term<BK>(base, ms, P.s[0], m3, kt, ti * BM, bar);
          if (NS == 2 && ns == 2) tma_term<BK>(base + BUF_BYTES, ms + 1, P.s[1], m3, kt, ti * BM, bar);
          if (!same) {
            tma_term<BK>(base + NS * BUF_BYTES, mt, tt[0], m3, kt, tj * BN, bar);
            if (NT == 2 && nt == 2) tma_term<BK>(base + (NS + 1) * BUF_BYTES, mt + 1, tt[1], m3, kt, tj * BN, bar);
          }
        }
      }
      kstep = __shfl_sync(0xffffffffu, kstep, 0);
    }
    return;
  }

  // ===================== consumer warpgroups =====================
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(wst::CONSUMER_REGS));
  const int ctid = tid - PRODUCERS;
  const int cw = warp - PRODUCERS / 32;
  const int wm = cw >> 2, wn = cw & 3;
  const int g = lane >> 2, q = lane & 3;
  // per-lane fragment offsets inside an operand k-block (see the header note):
  // [k-step parity][block parity]; the rest is compile-time
  uint32_t in_atom[2][2];
#pragma unroll
  for (int jp = 0; jp < 2; ++jp)
#pragma unroll
    for (int rp = 0; rp < 2; ++rp) {
      const int x = 2 * q + jp;
      const int chunk = (rp * 4 + (g >> 1)) ^ x;
      in_atom[jp][rp] = x * 128 + chunk * 16 + (g & 1) * 8;
    }
  // Diagonal SYRK tiles: only the 8x8 blocks on or below the diagonal are
  // computed, and the warps take their 64x32 sub-tiles in a permuted order so
  // the two warps sharing an SM sub-partition (cw, cw + 4) split the lower
  // triangle's 136 blocks 32/32/36/36 instead of 64/64/64/64 (the DMMA pipe is
  // per sub-partition): a diagonal tile costs ~56 % of a full one.
  // (wm, wn) of consumer warp cw on diagonal tiles, packed: wm = {1,1,0,1,0,0,1,0},
  // wn = {0,1,0,2,2,3,3,1}
  const int dwm = (75 >> cw) & 1, dwn = (32388 >> (2 * cw)) & 3;
  const uint32_t smem0 = smem_u32(smem);
  int kstep = 0;
  for (int it = 0;; ++it) {
    const int slot = it % kSlots;
    mbar_wait(&tfull[slot], (it / kSlots) & 1);
    const int tile = tinfo[slot];
    if (tile >= args.total_tiles) break;
    TileInfo tl;
    tl.pi = tdec[slot][0];
    tl.ti = tdec[slot][1];
    tl.tj = tdec[slot][2];
    const PD& P = *reinterpret_cast<const PD*>(pdesc_raw + slot * sizeof(PD));
    const bool same = P.kind == kSyrk && tl.ti == tl.tj;
    const int KT = (P.m + BK - 1) / BK;
    double acc[WTM][WTN][2];
#pragma unroll
    for (int r = 0; r < WTM; ++r)
#pragma unroll
      for (int c = 0; c < WTN; ++c) acc[r][c][0] = acc[r][c][1] = 0.0;
    const int twm = same ? dwm : wm, twn = same ? dwn : wn;
    const uint32_t abase = (twm * (WTM / 2)) * BK * 128, bbase = (twn * (WTN / 2)) * BK * 128;
    const uint32_t bsel = same ? 0u : (uint32_t)(NS * BUF_BYTES);
    // second terms: S1 / T1 one buffer after S0 / T0, added with their signs
    const bool two_a = NS == 2 && P.ns == 2;
    const bool two_b = same ? two_a : (NT == 2 && P.kind != kSyrk && P.nt == 2);
    const double sa = two_a ? P.s[1].sign : 0.0;
    const double sb = same ? sa : (two_b ? P.t[1].sign : 0.0);
    // OFF: the warp's 8x8 block (r, c) is computed iff c < r + OFF (on or below the
    // diagonal of a diagonal tile: OFF = 8 wm - 4 wn + 1); 99 = every block, -99 = none.
    // A compile-time pattern per warp role: predicated-off DMMAs would still spend
    // their issue slots, branch-free unrolled code skips them.
    auto mainloop = [&](auto off_tag) {
      constexpr int OFF = decltype(off_tag)::value;
      for (int kt = 0; kt < KT; ++kt, ++kstep) {
        const int s = kstep % STAGES;
        mbar_wait(&full[s], (kstep / STAGES) & 1);
        const uint32_t As = smem0 + s * STAGE_BYTES + abase;
        const uint32_t Bs = smem0 + s * STAGE_BYTES + bsel + bbase;
#pragma unroll
        for (int j = 0; j < BK / 4; ++j) {
          double a[WTM], b[WTN];
#pragma unroll
          for (int r = 0; r < WTM; ++r)
            a[r] = lds64(As + in_atom[j & 1][r & 1] + (r >> 1) * BK * 128 + (j >> 1) * 1024);
#pragma unroll
          for (int c = 0; c < WTN; ++c)
            b[c] = lds64(Bs + in_atom[j & 1][c & 1] + (c >> 1) * BK * 128 + (j >> 1) * 1024);
          if (NS == 2 && two_a) {
#pragma unroll
            for (int r = 0; r < WTM; ++r)
              a[r] = fma(sa, lds64(As + BUF_BYTES + in_atom[j & 1][r & 1] + (r >> 1) * BK * 128 + (j >> 1) * 1024),
                         a[r]);
          }
          if ((NS == 2 || NT == 2) && two_b) {
#pragma unroll
            for (int c = 0; c < WTN; ++c)
              b[c] = fma(sb, lds64(Bs + BUF_BYTES + in_atom[j & 1][c & 1] + (c >> 1) * BK * 128 + (j >> 1) * 1024),
                         b[c]);
          }
#pragma unroll
          for (int r = 0; r < WTM; ++r)
#pragma unroll
            for (int c = 0; c < WTN; ++c)
              if (c < r + OFF) dmma_ws(acc[r][c], a[r], b[c]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    };
    const int off = 8 * twm - 4 * twn + 1;
    if (!same || off >= WTN)
      mainloop(std::integral_constant<int, 99>());
    else if (off <= 1 - WTM)
      mainloop(std::integral_constant<int, -99>());
    else if (off == 1)
      mainloop(std::integral_constant<int, 1>());
    else
      mainloop(std::integral_constant<int, -3>());   // the permuted map's only other pattern
    ws_epilogue(args, P, tl, acc, twm, twn, g, q, ctid);
    __syncwarp();
    if (lane == 0) mbar_arrive(&tempty[slot]);
  }
}

// ---- device-resident descriptors (BatchArgsG) ----
namespace {
struct DescEntry {
  std::vector<unsigned char> host;  // exact bytes (descriptors + tile table) for hit checks
  void* dev = nullptr;
  uint64_t last_use = 0;
  // used by a launch recorded into a CUDA graph: the graph keeps the device
  // pointer for as long as it lives, so the entry is never evicted
  bool pinned = false;
  size_t payload_bytes = 0;
};
struct DescCache {
  std::unordered_map<uint64_t, DescEntry> map;
  size_t bytes = 0;
  uint64_t clock = 0;
};
std::mutex& desc_mutex() {
  static std::mutex mu;
  return mu;
}
DescCache& desc_cache() {  // caller holds desc_mutex()
  static std::map<int, DescCache> per_device;
  int dev = 0;
  cudaGetDevice(&dev);
  return per_device[dev];
}
uint64_t blob_hash(const unsigned char* p, size_t n) {  // 64-bit words (blobs are 8-byte multiples)
  uint64_t h = 1469598103934665603ull ^ n;
  const uint64_t* w = reinterpret_cast<const uint64_t*>(p);
  for (size_t i = 0; i < n / 8; ++i) {
    h ^= w[i] + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    h *= 1099511628211ull;
  }
  return h;
}
}  // namespace

// Device copy of a launch's descriptor blob, cached by content (repeated plans
// hit it; entries used while a graph is captured are pinned for the graph's
// lifetime).  cudaErrorNotReady: not resident and the stream is capturing.
// `sig` identifies the content (hashed, compared on a hit); `build` makes the
// device payload only on a miss (the TMA launches' tensor maps are expensive to
// encode: ~20k for a c2 leaf group).
template <typename Build>
static cudaError_t resident_blob_sig(std::vector<unsigned char>& sig, Build build, cudaStream_t s, void** dev) {
  std::lock_guard<std::mutex> lock(desc_mutex());
  DescCache& cache = desc_cache();
  const uint64_t key = blob_hash(sig.data(), sig.size());
  auto it = cache.map.find(key);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  const bool capturing = cs != cudaStreamCaptureStatusNone;
  if (it == cache.map.end() || it->second.host != sig) {
    if (capturing) return cudaErrorNotReady;  // no uploads inside a capture
    if (it != cache.map.end()) {  // hash collision: replace
      if (it->second.pinned) return cudaErrorNotReady;  // a live graph holds the colliding entry: narrow batches
      cudaFree(it->second.dev);
      cache.bytes -= it->second.host.size() + it->second.payload_bytes;
      cache.map.erase(it);
    }
    // evict least recently used unpinned entries beyond the budget (256 MB;
    // ATA_DESC_CACHE_KB overrides it, read on every miss)
    const char* lim_env = std::getenv("ATA_DESC_CACHE_KB");
    const size_t limit = lim_env ? (size_t)std::atoll(lim_env) << 10 : (size_t)256 << 20;
    while (cache.bytes + sig.size() > limit) {
      auto lru = cache.map.end();
      for (auto j = cache.map.begin(); j != cache.map.end(); ++j)
        if (!j->second.pinned && (lru == cache.map.end() || j->second.last_use < lru->second.last_use)) lru = j;
      if (lru == cache.map.end()) break;  // everything left is held by graphs
      cudaDeviceSynchronize();  // the evicted buffer may be in use by queued work on any stream
      cudaFree(lru->second.dev);
      cache.bytes -= lru->second.host.size() + lru->second.payload_bytes;
      cache.map.erase(lru);
    }
    std::vector<unsigned char> payload;
    if (cudaError_t e = build(payload); e != cudaSuccess) return e;
    DescEntry ent;
    cudaError_t e = cudaMalloc(&ent.dev, payload.size());
    if (e != cudaSuccess) return e;
    e = cudaMemcpy(ent.dev, payload.data(), payload.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return e;
    ent.host = std::move(sig);
    cache.bytes += ent.host.size() + payload.size();
    ent.payload_bytes = payload.size();
    it = cache.map.emplace(key, std::move(ent)).first;
  }
  it->second.last_use = ++cache.clock;
  if (capturing) it->second.pinned = true;
  *dev = it->second.dev;
  return cudaSuccess;
}

static cudaError_t resident_blob(std::vector<unsigned char>& blob, cudaStream_t s, void** dev) {
  std::vector<unsigned char> copy;
  return resident_blob_sig(
      blob,
      [&](std::vector<unsigned char>& out) {
        out = blob;
        return cudaSuccess;
      },
      s, dev);
}

cudaError_t launch_batch_f64_global(DProdT<double, kNarrowDests>* prods, int count, double alpha, int* sync,
                                    cudaStream_t s) {
  using namespace ws64;
  long long total = 0;
  int ns = 1, nt = 1;
  for (int i = 0; i < count; ++i) {
    auto& p = prods[i];
    p.tn = (p.n + BM - 1) / BM;
    p.tk = (p.k + BN - 1) / BN;
    p.tile_begin = (int)total;
    total += p.kind == kSyrk ? (long long)p.tn * (p.tn + 1) / 2 : (long long)p.tn * p.tk;
    ns = max(ns, p.ns);
    if (p.kind != kSyrk) nt = max(nt, p.nt);
    for (int d = 0; d < p.nd; ++d) p.d[d].sem = -1;  // region-free by contract
  }
  if (total <= 0) return cudaSuccess;
  if (total > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  const size_t dbytes = sizeof(DProdT<double, kNarrowDests>) * (size_t)count;
  std::vector<unsigned char> blob(dbytes + ((sizeof(int) * (size_t)total + 7) & ~size_t(7)), 0);
  std::memcpy(blob.data(), prods, dbytes);
  int* tp = reinterpret_cast<int*>(blob.data() + dbytes);
  for (int i = 0; i < count; ++i) {
    const auto& p = prods[i];
    const long long nt_i = p.kind == kSyrk ? (long long)p.tn * (p.tn + 1) / 2 : (long long)p.tn * p.tk;
    for (long long t = 0; t < nt_i; ++t) tp[p.tile_begin + t] = i;
  }
  void* dev_blob = nullptr;
  if (cudaError_t e = resident_blob(blob, s, &dev_blob); e != cudaSuccess) return e;
  BatchArgsGlobal64 a;
  std::memset(&a, 0, sizeof(a));
  a.count = count;
  a.total_tiles = (int)total;
  a.alpha = alpha;
  // dynamic tile queue: the group mixes long (diagonal / merged) and short products
  a.dynamic = sync != nullptr;
  a.sync = sync;
  a.n_sync = 1;
  if (a.dynamic) {
    cudaError_t e = cudaMemsetAsync(sync, 0, sizeof(int), s);
    if (e != cudaSuccess) return e;
  }
  { const char* e = std::getenv("ATA_DBG"); a.dbg = e ? std::atoi(e) : 0; }
  a.gp = reinterpret_cast<const DProdT<double, kNarrowDests>*>(dev_blob);
  a.tile_prod = reinterpret_cast<const int*>(reinterpret_cast<const unsigned char*>(dev_blob) + dbytes);
#ifndef WSG_BK
#define WSG_BK 16   // k-block rows of single-term device-descriptor batches
#endif
  if (ns == 1 && nt == 1) return ws_kernel_launch<WSG_BK, 1, 1>(a, total, s);
  if (ns == 2 && nt == 1) return ws_kernel_launch<WS2_BK, 2, 1>(a, total, s);
  if (ns == 1 && nt == 2) return ws_kernel_launch<WS2_BK, 1, 2>(a, total, s);
  return ws_kernel_launch<WS2_BK, 2, 2>(a, total, s);
}
cudaError_t launch_batch_f64_ws_narrow(const BatchArgsNarrow64& a, cudaStream_t s) { return launch_ws_any(a, s); }

// ---- TMA-fed launches (prod_f64_tma_kernel) ----
static PFN_cuTensorMapEncodeTiled_v12000 f64_encoder() {
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

// A window as [panels][rows][16 doubles] (panel stride 128 B), boxes of
// [BM/16 panels][BK rows][16] with the 128-byte swizzle; rows and panels
// outside the window are zero-filled.
static bool f64_map_term(CUtensorMap* map, const DTerm<double>& t, int bk) {
  auto enc = f64_encoder();
  if (enc == nullptr) return false;
  cuuint64_t dims[3] = {16, (cuuint64_t)t.rows, (cuuint64_t)(t.cols / 16)};
  cuuint64_t strides[2] = {(cuuint64_t)t.ld * 8, 128};
  cuuint32_t box[3] = {16, (cuuint32_t)bk, wst::PANELS};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(t.p), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D map of a window with an even pitch and any 8-byte alignment: based at
// the window start rounded down to 16 bytes (col0 = 0 or 1 element before it),
// extent [col0 + cols, rounded up to even][rows], boxes [BK rows][16 doubles],
// 128-byte swizzle; everything past the window's last row (the contraction) is
// zero-filled, columns past it only reach truncated output columns
static bool f64_map_term2d(CUtensorMap* map, const DTerm<double>& t, int bk) {
  auto enc = f64_encoder();
  if (enc == nullptr) return false;
  const uintptr_t p = reinterpret_cast<uintptr_t>(t.p);
  const uintptr_t base = p & ~uintptr_t(15);
  const cuuint64_t col0 = (p - base) / 8;
  // the inner extent must be a whole number of 16-byte units (an odd one faults
  // the TMA unit -- measured): round up; the extra column lies inside the even
  // pitch and only feeds output columns the epilogue truncates
  const cuuint64_t width = col0 + (cuuint64_t)t.cols;
  cuuint64_t dims[2] = {width + (width & 1), (cuuint64_t)t.rows};
  cuuint64_t strides[1] = {(cuuint64_t)t.ld * 8};
  cuuint32_t box[2] = {16, (cuuint32_t)bk};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, reinterpret_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool tma_term3d(const DTerm<double>& t) {
  return (reinterpret_cast<uintptr_t>(t.p) & 15) == 0 && (t.ld & 1) == 0 && t.cols % 16 == 0 && t.cols >= 16;
}
// (a box may not start 8 bytes into a 16-byte unit -- measured: the load
// faults -- so windows must start 16-byte aligned; with even pitches that is
// an even column offset, which every window of the reference trees has once A
// and the scratch buffers use even pitches)
static bool tma_term_ok(const DTerm<double>& t, bool first) {
  return (reinterpret_cast<uintptr_t>(t.p) & 15) == 0 && (t.ld & 1) == 0 && t.rows >= 1 && t.cols >= 1 &&
         (!first || t.sign == 1.0);
}

bool f64_tma_eligible(const DProdT<double, kNarrowDests>* prods, int count) {
  static const int mode = [] {
    const char* e = std::getenv("ATA_F64_TMA");
    return e ? std::atoi(e) : 1;
  }();
  if (mode == 0 || f64_encoder() == nullptr) return false;
  // an odd window width is rounded up to a whole 16-byte unit by the 2-D map, so the
  // TMA unit delivers the element after the window's last column instead of the zero
  // of the reference's zero-extension: harmless when that column lies beyond the
  // product's extent (the epilogue truncates it), wrong when the window is narrower
  // than the product (odd Strassen quadrants) -- those take the cp.async kernel
  auto width_ok = [](const DTerm<double>& t, int extent) { return (t.cols & 1) == 0 || t.cols >= extent; };
  for (int i = 0; i < count; ++i) {
    const auto& p = prods[i];
    if (p.ns < 1 || p.ns > 2 || !tma_term_ok(p.s[0], true) || (p.ns == 2 && !tma_term_ok(p.s[1], false)))
      return false;
    if (p.kind == kSyrk && p.ns != 1) return false;
    if (p.kind != kSyrk && (p.nt < 1 || p.nt > 2 || !tma_term_ok(p.t[0], true) ||
                            (p.nt == 2 && !tma_term_ok(p.t[1], false))))
      return false;
    for (int j = 0; j < p.ns; ++j)
      if (!width_ok(p.s[j], p.n)) return false;
    if (p.kind != kSyrk)
      for (int j = 0; j < p.nt; ++j)
        if (!width_ok(p.t[j], p.k)) return false;
  }
  return true;
}

template <int BK, int NS, int NT>
static cudaError_t tma_kernel_launch(const TmaBatch64& a, long long total, cudaStream_t s) {
  constexpr int STAGES = wst::stages<BK, NS, NT>();
  const size_t smem = 1024 + (size_t)STAGES * wst::stage_bytes<BK, NS, NT>() + (2 * STAGES + 2 * 3) * sizeof(uint64_t) +
                      4 * sizeof(int);
  auto kern = prod_f64_tma_kernel<BK, NS, NT>;
  static std::atomic<unsigned long long> attr_set{0};
  if (cudaError_t e = ata::set_smem_attr(kern, smem, attr_set); e != cudaSuccess) return e;
  const int grid = (int)(total < num_sms() ? total : num_sms());
  kern<<<grid, ws64::THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

// ---- riding operand sums: host side ----
static bool ride_win_ok(const void* p, long long ld, int rows, int cols) {
  return rows >= 0 && cols >= 0 && (cols & 1) == 0 && (ld & 1) == 0 && ld < 0x7fffffffLL &&
         (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}
bool f64_ride_eligible(const EwArgs<double>& a) {
  if (a.lower || a.nsrc < 1 || a.nsrc > 4 || a.ndst < 1 || a.ndst > 5 || a.rows < 1 || a.cols < 2 || (a.cols & 1))
    return false;
  for (int q = 0; q < a.nsrc; ++q)   // sources: one common pitch (the quadrants of one window)
    if (!ride_win_ok(a.src[q].p, a.src[q].ld, a.src[q].rows, a.src[q].cols) || a.src[q].ld != a.src[0].ld)
      return false;
  for (int j = 0; j < a.ndst; ++j)   // outputs: full-extent blocks with one common pitch
    if (!ride_win_ok(a.dst[j].p, a.dst[j].ld, a.dst[j].rows, a.dst[j].cols) || a.dst[j].ld != a.dst[0].ld ||
        a.dst[j].rows != a.rows || a.dst[j].cols != a.cols || (unsigned)a.dst[j].coef > 255u)
      return false;
  return true;
}
namespace {
struct Span {   // bounding address interval of a window (conservative for strided windows)
  uintptr_t lo, hi;
};
template <typename W>
Span span_of(const W& w) {
  if (w.rows <= 0 || w.cols <= 0) return {0, 0};
  const uintptr_t lo = reinterpret_cast<uintptr_t>(w.p);
  return {lo, lo + ((uintptr_t)(w.rows - 1) * (uintptr_t)w.ld + (uintptr_t)w.cols) * sizeof(double)};
}
bool overlap(Span a, Span b) { return a.lo < a.hi && b.lo < b.hi && a.lo < b.hi && b.lo < a.hi; }
// b conflicts with a (a earlier): b reads what a writes, or b writes what a reads or writes
bool ride_conflict(const EwArgs<double>& a, const EwArgs<double>& b) {
  for (int j = 0; j < b.ndst; ++j) {
    for (int q = 0; q < a.nsrc; ++q)
      if (overlap(span_of(b.dst[j]), span_of(a.src[q]))) return true;
    for (int e = 0; e < a.ndst; ++e)
      if (overlap(span_of(b.dst[j]), span_of(a.dst[e]))) return true;
  }
  for (int q = 0; q < b.nsrc; ++q)
    for (int e = 0; e < a.ndst; ++e)
      if (overlap(span_of(b.src[q]), span_of(a.dst[e]))) return true;
  return false;
}
}  // namespace

// The riding nodes must be independent of the launch's products: they may not
// write anything a product reads or writes, nor read anything a product writes
// (checked on bounding intervals; the planner guarantees it, this is the guard).
static bool ride_independent(const EwArgs<double>* ride, int n_ride, const DProdT<double, kNarrowDests>* prods,
                             int count) {
  for (int i = 0; i < n_ride; ++i) {
    const EwArgs<double>& a = ride[i];
    for (int pi = 0; pi < count; ++pi) {
      const auto& p = prods[pi];
      for (int j = 0; j < a.ndst; ++j) {
        const Span d = span_of(a.dst[j]);
        for (int q = 0; q < p.ns; ++q)
          if (overlap(d, span_of(p.s[q]))) return false;
        for (int q = 0; q < (p.kind == kSyrk ? 0 : p.nt); ++q)
          if (overlap(d, span_of(p.t[q]))) return false;
        for (int e = 0; e < p.nd; ++e)
          if (overlap(d, span_of(p.d[e]))) return false;
      }
      for (int q = 0; q < a.nsrc; ++q)
        for (int e = 0; e < p.nd; ++e)
          if (overlap(span_of(a.src[q]), span_of(p.d[e]))) return false;
    }
  }
  return true;
}

// RideNodes of a ride (phases by dependency among the nodes, chunk prefix);
// false when the ride cannot run inside the launch (the caller then runs the
// nodes as ordinary combo4 launches first).
static bool build_ride(const EwArgs<double>* ride, int n_ride, std::vector<RideNode>& out, int& chunks,
                       int& phases) {
  out.clear();
  chunks = 0;
  phases = 0;
  int phase = 0, phase_first = 0, phase_chunks = 0, prev_phase_chunks = 0;
  for (int i = 0; i < n_ride; ++i) {
    const EwArgs<double>& a = ride[i];
    if (!f64_ride_eligible(a)) return false;
    bool dep = false;
    for (int e = phase_first; e < i && !dep; ++e) dep = ride_conflict(ride[e], a);
    if (dep) {
      ++phase;
      phase_first = i;
      prev_phase_chunks = phase_chunks;
      phase_chunks = 0;
      // (a node also conflicting with phases before the previous one is covered:
      // finishing phase p - 1 implies every earlier phase finished)
    }
    if (phase >= kMaxRidePhases) return false;
    RideNode n;
    std::memset(&n, 0, sizeof(n));
    for (int q = 0; q < a.nsrc; ++q) {
      n.src[q] = a.src[q].p;
      n.srows[q] = a.src[q].rows;
      n.scols[q] = a.src[q].cols;
    }
    for (int j = 0; j < a.ndst; ++j) {
      n.dst[j] = a.dst[j].p;
      n.codes |= (unsigned long long)(a.dst[j].coef & 255) << (8 * j);
    }
    n.sld = (int)a.src[0].ld;
    n.dld = (int)a.dst[0].ld;
    n.nsrc = a.nsrc;
    n.ndst = a.ndst;
    n.rows = a.rows;
    n.cp = a.cols / 2;
    n.strips = (n.cp + 31) / 32;
    n.chunk_begin = chunks;
    n.phase = phase;
    n.wait_chunks = phase > 0 ? prev_phase_chunks : 0;
    const long long c = (long long)n.strips * ((n.rows + kRideRows - 1) / kRideRows);
    if (chunks + c > 0x3fffffffLL) return false;
    chunks += (int)c;
    phase_chunks += (int)c;
    out.push_back(n);
  }
  phases = phase + 1;
  return !out.empty();
}

cudaError_t launch_batch_f64_tma(DProdT<double, kNarrowDests>* prods, int count, double alpha, int* sync,
                                 long long sync_ints, cudaStream_t s, const EwArgs<double>* ride, int n_ride) {
  using namespace ws64;
  long long total = 0;
  for (int i = 0; i < count; ++i) {
    auto& p = prods[i];
    p.tn = (p.n + BM - 1) / BM;
    p.tk = (p.k + BN - 1) / BN;
    p.tile_begin = (int)total;
    total += p.kind == kSyrk ? (long long)p.tn * (p.tn + 1) / 2 : (long long)p.tn * p.tk;
  }
  if (total <= 0) return n_ride > 0 ? cudaErrorNotSupported : cudaSuccess;
  if (total > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  // destination regions (DDest.sem = batch-local region id, 1-based; 0 = none):
  // per-tile turn counters at sync[1..], as in launch_ws
  const int nreg = count * kNarrowDests;
  std::vector<int> rbase(nreg, -1), rld(nreg, 0), rrows(nreg, 0), rseen(nreg, 0);
  for (int i = 0; i < count; ++i)
    for (int d = 0; d < prods[i].nd; ++d) {
      const int rg = prods[i].d[d].sem;
      if (rg <= 0 || rg > nreg) continue;
      rld[rg - 1] = max(rld[rg - 1], prods[i].tk);
      rrows[rg - 1] = max(rrows[rg - 1], prods[i].tn);
    }
  long long n_sync = 1;
  for (int r = 0; r < nreg; ++r)
    if (rld[r] > 0) {
      rbase[r] = (int)n_sync;
      n_sync += (long long)rld[r] * rrows[r];
    }
  for (int i = 0; i < count; ++i)
    for (int d = 0; d < prods[i].nd; ++d) {
      DDest<double>& D = prods[i].d[d];
      const int rg = D.sem;
      if (rg <= 0 || rg > nreg) {
        D.sem = -1;
        continue;
      }
      D.sem = rbase[rg - 1];
      D.sem_ld = rld[rg - 1];
      D.turn = rseen[rg - 1]++;
    }
  // dynamic tile queue (tiles still start in increasing order): groups mix
  // tiles of very different contraction lengths (merged diagonal SYRKs, tail
  // chunks); ATA_F64_TMA_STATIC=1 selects the static round-robin
  static const bool force_static = std::getenv("ATA_F64_TMA_STATIC") != nullptr;
  const bool dynamic = n_sync > 1 || (sync != nullptr && sync_ints >= 1 && !force_static);
  if (dynamic && (sync == nullptr || n_sync > sync_ints)) return cudaErrorInvalidValue;
  // riding operand sums: their chunk queue and per-phase counts follow the turn counters
  std::vector<RideNode> rnodes;
  int ride_chunks = 0, ride_phases = 0;
  if (n_ride > 0) {
    const char* why = nullptr;
    if (sync == nullptr) why = "no sync buffer";
    else if (!build_ride(ride, n_ride, rnodes, ride_chunks, ride_phases)) why = "ineligible node (or too many phases)";
    else if (n_sync + 1 + ride_phases > sync_ints) why = "sync buffer too small";
    else if (!ride_independent(ride, n_ride, prods, count)) why = "not independent of the products";
    if (why != nullptr) {
      static const bool dbg = std::getenv("ATA_RIDE_DEBUG") != nullptr;
      if (dbg) std::fprintf(stderr, "[ata] ride of %d nodes refused: %s\n", n_ride, why);
      return cudaErrorNotSupported;   // the caller runs the nodes as ordinary launches
    }
  }
  const size_t rbytes = sizeof(RideNode) * rnodes.size();
  // device blob: tensor maps (64-byte aligned), descriptors, tile -> product
  // table; identified by the descriptors themselves (the maps are a function of
  // them), so a repeated launch skips encoding its maps
  const size_t mbytes = sizeof(CUtensorMap) * 4 * (size_t)count;
  const size_t dbytes = sizeof(DProdT<double, kNarrowDests>) * (size_t)count;
  int ns = 1, nt = 1;
  for (int i = 0; i < count; ++i) {
    ns = max(ns, prods[i].ns);
    if (prods[i].kind != kSyrk) nt = max(nt, prods[i].nt);
  }
  const int bk = (ns == 1 && nt == 1) ? WST_BK : WST_BK2;   // the box rows of the kernel that runs
  bool map3d = true;   // every term a whole number of 16-column panels, 16-byte aligned
  for (int i = 0; i < count && map3d; ++i) {
    const auto& p = prods[i];
    for (int j = 0; j < p.ns; ++j) map3d = map3d && tma_term3d(p.s[j]);
    if (p.kind != kSyrk)
      for (int j = 0; j < p.nt; ++j) map3d = map3d && tma_term3d(p.t[j]);
  }
  std::vector<unsigned char> sig(dbytes + 4 * sizeof(int) + rbytes);
  std::memcpy(sig.data(), prods, dbytes);
  const int tail[4] = {0x544d4146, bk, map3d ? 1 : 0, (int)total};   // "TMA" tag: own hash domain
  std::memcpy(sig.data() + dbytes, tail, sizeof(tail));
  if (rbytes) std::memcpy(sig.data() + dbytes + sizeof(tail), rnodes.data(), rbytes);
  const size_t tbytes = (sizeof(int) * (size_t)total + 7) & ~size_t(7);
  auto build = [&](std::vector<unsigned char>& blob) -> cudaError_t {
    blob.assign(mbytes + dbytes + tbytes + rbytes, 0);
    if (rbytes) std::memcpy(blob.data() + mbytes + dbytes + tbytes, rnodes.data(), rbytes);
    CUtensorMap* maps = reinterpret_cast<CUtensorMap*>(blob.data());
    auto map_term = [&](CUtensorMap* m, const DTerm<double>& t) {
      return map3d ? f64_map_term(m, t, bk) : f64_map_term2d(m, t, bk);
    };
    for (int i = 0; i < count; ++i) {
      const auto& p = prods[i];
      for (int j = 0; j < p.ns; ++j)
        if (!map_term(&maps[4 * i + j], p.s[j])) return cudaErrorNotSupported;
      if (p.kind != kSyrk)
        for (int j = 0; j < p.nt; ++j)
          if (!map_term(&maps[4 * i + 2 + j], p.t[j])) return cudaErrorNotSupported;
    }
    std::memcpy(blob.data() + mbytes, prods, dbytes);
    int* tp = reinterpret_cast<int*>(blob.data() + mbytes + dbytes);
    for (int i = 0; i < count; ++i) {
      const auto& p = prods[i];
      const long long nt_i = p.kind == kSyrk ? (long long)p.tn * (p.tn + 1) / 2 : (long long)p.tn * p.tk;
      for (long long t = 0; t < nt_i; ++t) tp[p.tile_begin + t] = i;
    }
    return cudaSuccess;
  };
  void* dev = nullptr;
  if (cudaError_t e = resident_blob_sig(sig, build, s, &dev); e != cudaSuccess) return e;
  TmaBatch64 a;
  std::memset(&a, 0, sizeof(a));
  a.count = count;
  a.total_tiles = (int)total;
  a.alpha = alpha;
  a.sync = sync;
  a.n_sync = (int)n_sync;
  a.dynamic = dynamic ? 1 : 0;
  a.map3d = map3d ? 1 : 0;
  { const char* e = std::getenv("ATA_DBG"); a.dbg = e ? std::atoi(e) : 0; }
  a.maps = reinterpret_cast<const CUtensorMap*>(dev);
  a.gp = reinterpret_cast<const DProdT<double, kNarrowDests>*>(reinterpret_cast<const unsigned char*>(dev) + mbytes);
  a.tile_prod = reinterpret_cast<const int*>(reinterpret_cast<const unsigned char*>(dev) + mbytes + dbytes);
  if (!rnodes.empty()) {
    a.ride_nodes = (int)rnodes.size();
    a.ride_chunks = ride_chunks;
    a.ride = reinterpret_cast<const RideNode*>(reinterpret_cast<const unsigned char*>(dev) + mbytes + dbytes + tbytes);
    a.ride_sync = sync + n_sync;
  }
  if (dynamic || !rnodes.empty()) {
    const size_t ints = (size_t)n_sync + (rnodes.empty() ? 0 : 1 + (size_t)ride_phases);
    cudaError_t e = cudaMemsetAsync(sync, 0, ints * sizeof(int), s);
    if (e != cudaSuccess) return e;
  }
  if (ns == 1 && nt == 1) return tma_kernel_launch<WST_BK, 1, 1>(a, total, s);
  if (ns == 2 && nt == 1) return tma_kernel_launch<WST_BK2, 2, 1>(a, total, s);
  if (ns == 1 && nt == 2) return tma_kernel_launch<WST_BK2, 1, 2>(a, total, s);
  return tma_kernel_launch<WST_BK2, 2, 2>(a, total, s);
}


}  // namespace ata
