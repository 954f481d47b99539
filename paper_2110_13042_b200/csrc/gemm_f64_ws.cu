// FP64 generalized-product kernel, warp-specialised (sm_100a, DMMA.8x8x4).
//
// Same product semantics as gemm_f64.cu (fused zero-extended operand terms =
// Strassen pre-additions, strassen.py:195-203; fused truncated destinations =
// post-additions, strassen.py:238-275 / matrix.py:218-239; SYRK lower tiles,
// matrix.py:292-311).  Structure:
//
//   warp 0      producer: cp.async (16 B, or 8 B for odd pitches) of the
//               [BK x 128] operand windows into a STAGES-deep smem ring, with
//               zero-fill outside each term window; two-term operands are
//               combined in place by the producer once its copies land.
//               Completion is published through per-stage "full" mbarriers.
//   warps 1..8  consumers: 2 x 4 warps, 64 x 32 accumulator each (32 DMMA
//               8x8x4 blocks, fragments straight from the padded smem rows),
//               release a stage through its "empty" mbarrier; no CTA-wide
//               barrier in the main loop.  Epilogue writes up to four signed,
//               truncated destinations from registers.
//
// SYRK diagonal tiles load the operand panel once (both MMA operands read it).
#include "ata_common.cuh"

namespace ata {

namespace ws64 {
constexpr int BM = 128, BN = 128, BK = 16, LD = BM + 4;
constexpr int CONSUMERS = 8, PRODUCERS = 128, THREADS = CONSUMERS * 32 + PRODUCERS;
constexpr int PRODUCER_REGS = 40, CONSUMER_REGS = 232;  // setmaxnreg split of the 64K RF
constexpr int WTM = 8, WTN = 4;  // 64 x 32 per consumer warp
constexpr int BUF = BK * LD;     // doubles per operand buffer
constexpr int SMEM_BUDGET = 225 * 1024;
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

// One producer warp copies a BK x 128 window of term t (rows l0.., cols c0..).
template <bool VEC16>
__device__ __forceinline__ void ws_load(double* buf, const DTerm<double>& t, int l0, int c0, int lane) {
  using namespace ws64;
  if (VEC16) {
#pragma unroll 8
    for (int i = 0; i < BK * (BM / 2) / PRODUCERS; ++i) {
      const int id = lane + i * PRODUCERS;
      const int r = id >> 6;            // BM/2 = 64 chunks per row
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
#pragma unroll 8
    for (int i = 0; i < BK * BM / PRODUCERS; ++i) {
      const int id = lane + i * PRODUCERS;
      const int r = id >> 7;
      const int c = id & 127;
      const int gl = l0 + r, gc = c0 + c;
      const int bytes = (gl < t.rows && gc < t.cols) ? 8 : 0;
      const double* src = bytes ? t.p + (long long)gl * t.ld + gc : t.p;
      cp_async_8(buf + r * LD + c, src, bytes);
    }
  }
}

template <bool VEC16>
__device__ __forceinline__ void ws_combine(double* x, const double* y, double sign, int lane) {
  using namespace ws64;
  if (VEC16) {
#pragma unroll 8
    for (int i = 0; i < BK * (BM / 2) / PRODUCERS; ++i) {
      const int id = lane + i * PRODUCERS;
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
#pragma unroll 8
    for (int i = 0; i < BK * BM / PRODUCERS; ++i) {
      const int id = lane + i * PRODUCERS;
      const int r = id >> 7;
      const int c = id & 127;
      x[r * LD + c] = fma(sign, y[r * LD + c], x[r * LD + c]);
    }
  }
}

__device__ __forceinline__ bool vec16_ok(const DTerm<double>& t) {
  return ((reinterpret_cast<uintptr_t>(t.p) & 15) == 0) && ((t.ld & 1) == 0);
}

template <int NS, int NT, int STAGES>
__global__ void __launch_bounds__(ws64::THREADS, 1)
    prod_f64_ws_kernel(const __grid_constant__ BatchArgs<double> args) {
  using namespace ws64;
  constexpr int STAGE = (NS + NT) * BUF;
  extern __shared__ __align__(128) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  // ---- locate product and output tile ----
  const int tile = blockIdx.x;
  int pi = 0;
  while (pi + 1 < args.count && tile >= args.p[pi + 1].tile_begin) ++pi;
  const DProd<double>& P = args.p[pi];
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
  const int i0 = ti * BM, j0 = tj * BN;
  const bool syrk = (P.kind == kSyrk);
  const bool same = syrk && ti == tj;  // diagonal SYRK tile: one operand panel
  const int ns = P.ns, nt = syrk ? 1 : P.nt;
  const int KT = (P.m + BK - 1) / BK;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], PRODUCERS);
      mbar_init(&empty[s], CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (tid < PRODUCERS) {
    // ===================== producer warpgroup =====================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PRODUCER_REGS));
    const int lane = tid;  // producer thread index
    const DTerm<double>& S0 = P.s[0];
    const DTerm<double>& S1 = P.s[1];
    const DTerm<double>& T0 = syrk ? P.s[0] : P.t[0];
    const DTerm<double>& T1 = P.t[1];
    const bool vs = vec16_ok(S0) && (ns < 2 || vec16_ok(S1));
    const bool vt = vec16_ok(T0) && (nt < 2 || vec16_ok(T1));
    const bool comb = (NS == 2 && ns == 2) || (NT == 2 && nt == 2);
    auto issue = [&](int kt) {
      double* base = smem + (kt % STAGES) * STAGE;
      const int l0 = kt * BK;
      if (vs) ws_load<true>(base, S0, l0, i0, lane);
      else ws_load<false>(base, S0, l0, i0, lane);
      if (NS == 2 && ns == 2) {
        if (vs) ws_load<true>(base + BUF, S1, l0, i0, lane);
        else ws_load<false>(base + BUF, S1, l0, i0, lane);
      }
      if (!same) {
        double* tb = base + NS * BUF;
        if (vt) ws_load<true>(tb, T0, l0, j0, lane);
        else ws_load<false>(tb, T0, l0, j0, lane);
        if (NT == 2 && nt == 2) {
          if (vt) ws_load<true>(tb + BUF, T1, l0, j0, lane);
          else ws_load<false>(tb + BUF, T1, l0, j0, lane);
        }
      }
    };
    auto finish = [&](int kt) {  // combine two-term operands of stage kt, publish it
      double* base = smem + (kt % STAGES) * STAGE;
      if (NS == 2 && ns == 2) {
        if (vs) ws_combine<true>(base, base + BUF, S1.sign, lane);
        else ws_combine<false>(base, base + BUF, S1.sign, lane);
      }
      if (NT == 2 && nt == 2) {
        double* tb = base + NS * BUF;
        if (vt) ws_combine<true>(tb, tb + BUF, T1.sign, lane);
        else ws_combine<false>(tb, tb + BUF, T1.sign, lane);
      }
      mbar_arrive(&full[kt % STAGES]);
    };
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % STAGES;
      if (kt >= STAGES) mbar_wait(&empty[s], ((kt / STAGES) - 1) & 1);
      issue(kt);
      if (!comb) {
        mbar_arrive_cpasync(&full[s]);
      } else {
        cp_async_commit();
        if (kt >= 1) {
          cp_async_wait<1>();
          finish(kt - 1);
        }
      }
    }
    if (comb && KT >= 1) {
      cp_async_wait<0>();
      finish(KT - 1);
    }
    return;
  }

  // ===================== consumers =====================
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CONSUMER_REGS));
  const int cw = warp - PRODUCERS / 32;
  const int wm = cw >> 2, wn = cw & 3;  // 2 x 4 consumer warps
  const int g = lane >> 2, q = lane & 3;
  double acc[WTM][WTN][2];
#pragma unroll
  for (int r = 0; r < WTM; ++r)
#pragma unroll
    for (int c = 0; c < WTN; ++c) acc[r][c][0] = acc[r][c][1] = 0.0;

  const int aoff = wm * (WTM * 8) + g + q * LD;
  const int boff = (same ? 0 : NS * BUF) + wn * (WTN * 8) + g + q * LD;
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % STAGES;
    mbar_wait(&full[s], (kt / STAGES) & 1);
    const double* As = smem + s * STAGE + aoff;
    const double* Bs = smem + s * STAGE + boff;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double a[WTM], b[WTN];
#pragma unroll
      for (int r = 0; r < WTM; ++r) a[r] = As[kk * 4 * LD + r * 8];
#pragma unroll
      for (int c = 0; c < WTN; ++c) b[c] = Bs[kk * 4 * LD + c * 8];
#pragma unroll
      for (int r = 0; r < WTM; ++r)
#pragma unroll
        for (int c = 0; c < WTN; ++c) dmma_ws(acc[r][c], a[r], b[c]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---- epilogue: fused post-additions into up to four destinations ----
  const int nd = P.nd;
  const bool accumulate = P.accumulate != 0;
  for (int d = 0; d < nd; ++d) {
    const DDest<double>& D = P.d[d];
    const double scale = args.alpha * D.sign;
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
            const double2 o = *p2;
            v.x += o.x;
            v.y += o.y;
          }
          *p2 = v;
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cc = col + e;
            if (cc < D.cols && (!syrk || cc <= row)) {
              const double v = scale * acc[r][c][e];
              drow[cc] = accumulate ? drow[cc] + v : v;
            }
          }
        }
      }
    }
  }
}

template <int NS, int NT>
static cudaError_t launch_ws(BatchArgs<double> a, cudaStream_t s) {
  using namespace ws64;
  long long total = 0;
  for (int i = 0; i < a.count; ++i) {
    DProd<double>& p = a.p[i];
    p.tn = (p.n + BM - 1) / BM;
    p.tk = (p.k + BN - 1) / BN;
    p.tile_begin = (int)total;
    total += p.kind == kSyrk ? (long long)p.tn * (p.tn + 1) / 2 : (long long)p.tn * p.tk;
  }
  if (total <= 0) return cudaSuccess;
  if (total > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  a.total_tiles = (int)total;
  constexpr int STAGE_BYTES = (NS + NT) * BUF * 8;
  constexpr int STAGES = (SMEM_BUDGET - 1024) / STAGE_BYTES > 8 ? 8 : (SMEM_BUDGET - 1024) / STAGE_BYTES;
  static_assert(STAGES >= 2, "smem");
  const size_t smem = (size_t)STAGES * STAGE_BYTES + 2 * STAGES * sizeof(uint64_t);
  auto kern = prod_f64_ws_kernel<NS, NT, STAGES>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  kern<<<a.total_tiles, THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_batch_f64_ws(const BatchArgs<double>& a, cudaStream_t s) {
  int ns = 1, nt = 1;
  for (int i = 0; i < a.count; ++i) {
    ns = max(ns, a.p[i].ns);
    if (a.p[i].kind != kSyrk) nt = max(nt, a.p[i].nt);
  }
  if (ns == 1 && nt == 1) return launch_ws<1, 1>(a, s);
  if (ns == 2 && nt == 1) return launch_ws<2, 1>(a, s);
  if (ns == 1 && nt == 2) return launch_ws<1, 2>(a, s);
  return launch_ws<2, 2>(a, s);
}

}  // namespace ata
