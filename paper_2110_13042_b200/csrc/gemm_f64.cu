// FP64 generalized-product kernel for sm_100a (DMMA.8x8x4 tensor path).
//
// One launch executes a batch of write-disjoint "products"
//     D_d[:r_d, :c_d] (+)= sign_d * alpha * (sum_i s_i S_i)^T (sum_j t_j T_j)
// with up to two zero-extended operand terms per side (the Strassen
// pre-additions, strassen.py:195-203, fused into the tile load) and up to
// four truncated destinations (the Strassen post-additions, strassen.py:238-275
// via add_truncated matrix.py:218-239, fused into the epilogue).  A product
// with one term per side and one destination is the reference's leaf kernel
// naive_gemm_atb (matrix.py:269-289); kind kSyrk is naive_syrk_lower
// (matrix.py:292-311) restricted to lower-triangle tiles, masking the diagonal
// tiles on store so the strict upper triangle is never touched (ata.py:121-123).
//
// Both operands of A^T B on row-major A are "MN-major": the contraction runs
// down the rows.  Tiles are staged as [BK rows][BM cols] in shared memory with a
// +4 double pad, which makes the m8n8k4 fragment reads (lane -> (k=lane%4,
// col=lane/4)) conflict-free per half-warp.  Loads are cp.async (8 or 16 B,
// zero-filling outside the term window) in a multi-stage ring.  FP64 on B200 is
// 64 FMA/clk/SM through DMMA (measured 37.17 TF/s), so operand traffic is
// 8-16 B/clk/SM from L2 and TMA is not needed (odd leading dimensions -- config
// c2, 4097 columns -- also break TMA's 16-byte stride rule).
//
// The tile shape is a template (Cfg): warps x warp-tiles of 8x8 DMMA blocks.
#include <cstdlib>

#include "ata_common.cuh"

namespace ata {

template <int WARPS_M_, int WARPS_N_, int WTM_, int WTN_, int BK_, int STAGES_, int MINB_>
struct F64Cfg {
  static constexpr int WARPS_M = WARPS_M_, WARPS_N = WARPS_N_;
  static constexpr int WTM = WTM_, WTN = WTN_;  // 8x8 blocks per warp (rows, cols)
  static constexpr int BM = WARPS_M * WTM * 8, BN = WARPS_N * WTN * 8;
  static constexpr int BK = BK_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int LDA = BM + 4, LDB = BN + 4;  // padded smem rows (doubles)
};

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Load one BK x W window of a term (rows l0.., cols c0..) into buf (row pitch LD).
template <int BK, int W, int LD, int THREADS, bool VEC16>
__device__ __forceinline__ void load_term_f64(double* buf, const DTerm<double>& t, int l0, int c0,
                                              int tid) {
  if (VEC16) {
    constexpr int CH = BK * W / 2;  // 16-byte chunks
    static_assert(CH % THREADS == 0, "chunking");
#pragma unroll
    for (int i = 0; i < CH / THREADS; ++i) {
      const int id = tid + i * THREADS;
      const int r = id / (W / 2);
      const int c = (id % (W / 2)) * 2;
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
    constexpr int CH = BK * W;
    static_assert(CH % THREADS == 0, "chunking");
#pragma unroll
    for (int i = 0; i < CH / THREADS; ++i) {
      const int id = tid + i * THREADS;
      const int r = id / W;
      const int c = id % W;
      const int gl = l0 + r, gc = c0 + c;
      const int bytes = (gl < t.rows && gc < t.cols) ? 8 : 0;
      const double* src = bytes ? t.p + (long long)gl * t.ld + gc : t.p;
      cp_async_8(buf + r * LD + c, src, bytes);
    }
  }
}

// buf0 = buf0 + sign1 * buf1 over exactly the elements this thread loaded.
template <int BK, int W, int LD, int THREADS, bool VEC16>
__device__ __forceinline__ void combine_f64(double* buf0, const double* buf1, double sign1,
                                            int tid) {
  if (VEC16) {
    constexpr int CH = BK * W / 2;
#pragma unroll
    for (int i = 0; i < CH / THREADS; ++i) {
      const int id = tid + i * THREADS;
      const int r = id / (W / 2);
      const int c = (id % (W / 2)) * 2;
      double2* x = reinterpret_cast<double2*>(buf0 + r * LD + c);
      const double2 y = *reinterpret_cast<const double2*>(buf1 + r * LD + c);
      double2 v = *x;
      v.x = fma(sign1, y.x, v.x);
      v.y = fma(sign1, y.y, v.y);
      *x = v;
    }
  } else {
    constexpr int CH = BK * W;
#pragma unroll
    for (int i = 0; i < CH / THREADS; ++i) {
      const int id = tid + i * THREADS;
      const int r = id / W;
      const int c = id % W;
      buf0[r * LD + c] = fma(sign1, buf1[r * LD + c], buf0[r * LD + c]);
    }
  }
}

__device__ __forceinline__ bool term_vec16(const DTerm<double>& t) {
  return ((reinterpret_cast<uintptr_t>(t.p) & 15) == 0) && ((t.ld & 1) == 0);
}

// Largest ring depth <= CF::STAGES whose smem fits 227 KB (at least 2).
template <class CF, int NS, int NT>
__host__ __device__ constexpr int stages_for() {
  int s = CF::STAGES;
  while (s > 2 && (long)s * (NS * CF::BK * CF::LDA + NT * CF::BK * CF::LDB) * 8 > 227 * 1024) --s;
  return s;
}

template <class CF, int NS, int NT>
__global__ void __launch_bounds__(CF::THREADS, CF::MINB)
    prod_f64_kernel(const __grid_constant__ BatchArgs<double> args) {
  constexpr int BM = CF::BM, BN = CF::BN, BK = CF::BK, STAGES = stages_for<CF, NS, NT>();
  constexpr int LDA = CF::LDA, LDB = CF::LDB, THREADS = CF::THREADS;
  constexpr int WTM = CF::WTM, WTN = CF::WTN;
  constexpr int ABUF = BK * LDA, BBUF = BK * LDB;
  constexpr int STAGE = NS * ABUF + NT * BBUF;
  extern __shared__ __align__(128) double smem[];

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int wm = warp / CF::WARPS_N, wn = warp % CF::WARPS_N;

  // ---- locate product and output tile ----
  const int tile = blockIdx.x;
  int pi = 0;
  while (pi + 1 < args.count && tile >= args.p[pi + 1].tile_begin) ++pi;
  const DProd<double>& P = args.p[pi];
  const int local = tile - P.tile_begin;
  int ti, tj;
  if (P.kind == kSyrk) {
    // lower-triangular tile enumeration, row by row (BM == BN for SYRK configs)
    int r = (int)((sqrt(8.0 * (double)local + 1.0) - 1.0) * 0.5);
    while ((r + 1) * (r + 2) / 2 <= local) ++r;
    while (r * (r + 1) / 2 > local) --r;
    ti = r;
    tj = local - r * (r + 1) / 2;
  } else {
    // grouped raster: 8 tile-rows per group, column-major inside the group
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
  const int ns = P.ns, nt = syrk ? 1 : P.nt;
  const DTerm<double>& S0 = P.s[0];
  const DTerm<double>& S1 = P.s[1];
  const DTerm<double>& T0 = syrk ? P.s[0] : P.t[0];
  const DTerm<double>& T1 = P.t[1];
  const bool vs = term_vec16(S0) && (ns < 2 || term_vec16(S1));
  const bool vt = term_vec16(T0) && (nt < 2 || term_vec16(T1));

  auto load_stage = [&](int stage, int kt) {
    double* base = smem + stage * STAGE;
    const int l0 = kt * BK;
    if (vs) load_term_f64<BK, BM, LDA, THREADS, true>(base, S0, l0, i0, tid);
    else load_term_f64<BK, BM, LDA, THREADS, false>(base, S0, l0, i0, tid);
    if (NS == 2 && ns == 2) {
      if (vs) load_term_f64<BK, BM, LDA, THREADS, true>(base + ABUF, S1, l0, i0, tid);
      else load_term_f64<BK, BM, LDA, THREADS, false>(base + ABUF, S1, l0, i0, tid);
    }
    double* tb = base + NS * ABUF;
    if (vt) load_term_f64<BK, BN, LDB, THREADS, true>(tb, T0, l0, j0, tid);
    else load_term_f64<BK, BN, LDB, THREADS, false>(tb, T0, l0, j0, tid);
    if (NT == 2 && nt == 2) {
      if (vt) load_term_f64<BK, BN, LDB, THREADS, true>(tb + BBUF, T1, l0, j0, tid);
      else load_term_f64<BK, BN, LDB, THREADS, false>(tb + BBUF, T1, l0, j0, tid);
    }
  };

  double acc[WTM][WTN][2];
#pragma unroll
  for (int r = 0; r < WTM; ++r)
#pragma unroll
    for (int c = 0; c < WTN; ++c) acc[r][c][0] = acc[r][c][1] = 0.0;

  const int KT = (P.m + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    const int stage = kt % STAGES;
    cp_async_wait<STAGES - 2>();
    double* base = smem + stage * STAGE;
    if (NS == 2 && ns == 2) {
      if (vs) combine_f64<BK, BM, LDA, THREADS, true>(base, base + ABUF, S1.sign, tid);
      else combine_f64<BK, BM, LDA, THREADS, false>(base, base + ABUF, S1.sign, tid);
    }
    if (NT == 2 && nt == 2) {
      double* tb = base + NS * ABUF;
      if (vt) combine_f64<BK, BN, LDB, THREADS, true>(tb, tb + BBUF, T1.sign, tid);
      else combine_f64<BK, BN, LDB, THREADS, false>(tb, tb + BBUF, T1.sign, tid);
    }
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT) load_stage(nk % STAGES, nk);
      cp_async_commit();
    }
    const double* As = base + wm * (WTM * 8) + g;
    const double* Bs = base + NS * ABUF + wn * (WTN * 8) + g;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double a[WTM], b[WTN];
#pragma unroll
      for (int r = 0; r < WTM; ++r) a[r] = As[(kk * 4 + q) * LDA + r * 8];
#pragma unroll
      for (int c = 0; c < WTN; ++c) b[c] = Bs[(kk * 4 + q) * LDB + c * 8];
#pragma unroll
      for (int r = 0; r < WTM; ++r)
#pragma unroll
        for (int c = 0; c < WTN; ++c) dmma(acc[r][c], a[r], b[c]);
    }
  }
  cp_async_wait<0>();

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

template <class CF, int NS, int NT>
static cudaError_t launch_cfg(BatchArgs<double> a, cudaStream_t s) {
  // tile the batch for this configuration
  long long total = 0;
  for (int i = 0; i < a.count; ++i) {
    DProd<double>& p = a.p[i];
    p.tn = (p.n + CF::BM - 1) / CF::BM;
    p.tk = (p.k + CF::BN - 1) / CF::BN;
    p.tile_begin = (int)total;
    total += p.kind == kSyrk ? (long long)p.tn * (p.tn + 1) / 2 : (long long)p.tn * p.tk;
  }
  if (total <= 0) return cudaSuccess;
  if (total > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  a.total_tiles = (int)total;
  const size_t smem =
      (size_t)stages_for<CF, NS, NT>() * (NS * CF::BK * CF::LDA + NT * CF::BK * CF::LDB) * sizeof(double);
  auto kern = prod_f64_kernel<CF, NS, NT>;
  static std::atomic<unsigned long long> attr_set{0};  // per instantiation, per device
  if (cudaError_t e = ata::set_smem_attr(kern, smem, attr_set); e != cudaSuccess) return e;
  kern<<<a.total_tiles, CF::THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

// Configurations (square tiles: SYRK needs BM == BN).
using CfgA = F64Cfg<2, 4, 8, 4, 16, 4, 1>;   // 128x128, 8 warps of 64x32   (v0)
using CfgB = F64Cfg<4, 4, 4, 4, 16, 4, 1>;   // 128x128, 16 warps of 32x32
using CfgC = F64Cfg<2, 2, 4, 4, 16, 3, 4>;   // 64x64, 4 warps of 32x32, 4 CTAs/SM
using CfgD = F64Cfg<4, 4, 4, 4, 32, 3, 1>;   // 128x128, 16 warps, BK 32

static int pick_cfg() {
  static int cfg = -1;
  if (cfg < 0) {
    const char* e = std::getenv("ATA_F64_CFG");
    cfg = e ? std::atoi(e) : 4;
  }
  return cfg;
}

bool f64_supports_ordering() { return pick_cfg() == 4; }
bool f64_narrow_supported() { return pick_cfg() == 4; }
cudaError_t launch_batch_f64_ws_narrow(const BatchArgsNarrow64& a, cudaStream_t s);

template <int NS, int NT>
static cudaError_t launch_terms(const BatchArgs<double>& a, cudaStream_t s) {
  switch (pick_cfg()) {
    case 0: return launch_cfg<CfgA, NS, NT>(a, s);
    case 2: return launch_cfg<CfgC, NS, NT>(a, s);
    case 3: return launch_cfg<CfgD, NS, NT>(a, s);
    case 4: return launch_batch_f64_ws(a, s);
    default: return launch_cfg<CfgB, NS, NT>(a, s);
  }
}

// Narrow batches go to the persistent warp-specialised kernel in one launch
// (the executor forms them only when f64_narrow_supported()).
cudaError_t launch_batch_f64_narrow(const BatchArgsNarrow64& a, cudaStream_t s) {
  return launch_batch_f64_ws_narrow(a, s);
}

cudaError_t launch_batch_f64(const BatchArgs<double>& a, cudaStream_t s) {
  int ns = 1, nt = 1;
  for (int i = 0; i < a.count; ++i) {
    ns = max(ns, a.p[i].ns);
    if (a.p[i].kind != kSyrk) nt = max(nt, a.p[i].nt);
  }
  if (ns == 1 && nt == 1) return launch_terms<1, 1>(a, s);
  if (ns == 2 && nt == 1) return launch_terms<2, 1>(a, s);
  if (ns == 1 && nt == 2) return launch_terms<1, 2>(a, s);
  return launch_terms<2, 2>(a, s);
}

}  // namespace ata
