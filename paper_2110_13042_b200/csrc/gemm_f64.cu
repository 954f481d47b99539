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
// zero-filling outside the term window) in a multi-stage ring; FP64 on B200 is
// 64 FMA/clk/SM through DMMA, so operand bandwidth is ~8-16 B/clk/SM and TMA is
// not needed (and odd leading dimensions -- config c2, 4097 columns -- break
// TMA's 16-byte stride rule).
#include "ata_common.cuh"

namespace ata {

namespace f64cfg {
constexpr int BM = 128, BN = 128, BK = 16, LDS = BM + 4, THREADS = 256;
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Load one BK x 128 window of a term (rows l0.., cols c0..) into buf.
template <bool VEC16>
__device__ __forceinline__ void load_term_f64(double* buf, const DTerm<double>& t, int l0, int c0,
                                              int tid) {
  using namespace f64cfg;
  if (VEC16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = (tid >> 6) + 4 * i;
      const int c = (tid & 63) * 2;
      const int gl = l0 + r, gc = c0 + c;
      int bytes = 0;
      if (gl < t.rows) {
        const int left = t.cols - gc;
        bytes = left >= 2 ? 16 : (left == 1 ? 8 : 0);
      }
      const double* src = bytes ? t.p + (long long)gl * t.ld + gc : t.p;
      cp_async_16(buf + r * LDS + c, src, bytes);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = (tid >> 7) + 2 * i;
      const int c = tid & 127;
      const int gl = l0 + r, gc = c0 + c;
      const int bytes = (gl < t.rows && gc < t.cols) ? 8 : 0;
      const double* src = bytes ? t.p + (long long)gl * t.ld + gc : t.p;
      cp_async_8(buf + r * LDS + c, src, bytes);
    }
  }
}

// buf0 = buf0 + sign1 * buf1 over the elements this thread loaded.
template <bool VEC16>
__device__ __forceinline__ void combine_f64(double* buf0, const double* buf1, double sign1,
                                            int tid) {
  using namespace f64cfg;
  if (VEC16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = (tid >> 6) + 4 * i;
      const int c = (tid & 63) * 2;
      double2* x = reinterpret_cast<double2*>(buf0 + r * LDS + c);
      const double2 y = *reinterpret_cast<const double2*>(buf1 + r * LDS + c);
      double2 v = *x;
      v.x = fma(sign1, y.x, v.x);
      v.y = fma(sign1, y.y, v.y);
      *x = v;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = (tid >> 7) + 2 * i;
      const int c = tid & 127;
      buf0[r * LDS + c] = fma(sign1, buf1[r * LDS + c], buf0[r * LDS + c]);
    }
  }
}

__device__ __forceinline__ bool term_vec16(const DTerm<double>& t) {
  return ((reinterpret_cast<uintptr_t>(t.p) & 15) == 0) && ((t.ld & 1) == 0);
}

template <int NS, int NT, int STAGES>
__global__ void __launch_bounds__(f64cfg::THREADS, 1)
    prod_f64_kernel(const __grid_constant__ BatchArgs<double> args) {
  using namespace f64cfg;
  extern __shared__ __align__(128) double smem[];
  constexpr int BUF = BK * LDS;
  constexpr int STAGE = (NS + NT) * BUF;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps, warp tile 64 x 32

  // ---- locate product and output tile ----
  const int tile = blockIdx.x;
  int pi = 0;
  while (pi + 1 < args.count && tile >= args.p[pi + 1].tile_begin) ++pi;
  const DProd<double>& P = args.p[pi];
  const int local = tile - P.tile_begin;
  int ti, tj;
  if (P.kind == kSyrk) {
    // lower-triangular tile enumeration, row by row
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
    if (vs) load_term_f64<true>(base, S0, l0, i0, tid);
    else load_term_f64<false>(base, S0, l0, i0, tid);
    if (NS == 2 && ns == 2) {
      if (vs) load_term_f64<true>(base + BUF, S1, l0, i0, tid);
      else load_term_f64<false>(base + BUF, S1, l0, i0, tid);
    }
    double* tb = base + NS * BUF;
    if (vt) load_term_f64<true>(tb, T0, l0, j0, tid);
    else load_term_f64<false>(tb, T0, l0, j0, tid);
    if (NT == 2 && nt == 2) {
      if (vt) load_term_f64<true>(tb + BUF, T1, l0, j0, tid);
      else load_term_f64<false>(tb + BUF, T1, l0, j0, tid);
    }
  };

  double acc[8][4][2];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c][0] = acc[r][c][1] = 0.0;

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
      if (vs) combine_f64<true>(base, base + BUF, S1.sign, tid);
      else combine_f64<false>(base, base + BUF, S1.sign, tid);
    }
    if (NT == 2 && nt == 2) {
      double* tb = base + NS * BUF;
      if (vt) combine_f64<true>(tb, tb + BUF, T1.sign, tid);
      else combine_f64<false>(tb, tb + BUF, T1.sign, tid);
    }
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT) load_stage(nk % STAGES, nk);
      cp_async_commit();
    }
    const double* As = base;
    const double* Bs = base + NS * BUF;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double a[8], b[4];
      const int row = (kk * 4 + q) * LDS;
#pragma unroll
      for (int r = 0; r < 8; ++r) a[r] = As[row + wm * 64 + r * 8 + g];
#pragma unroll
      for (int c = 0; c < 4; ++c) b[c] = Bs[row + wn * 32 + c * 8 + g];
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) dmma(acc[r][c], a[r], b[c]);
    }
  }
  cp_async_wait<0>();

  // ---- epilogue: fused post-additions into up to four destinations ----
  const int nd = P.nd;
  for (int d = 0; d < nd; ++d) {
    const DDest<double>& D = P.d[d];
    const double scale = args.alpha * D.sign;
    const bool accumulate = P.accumulate != 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int row = i0 + wm * 64 + r * 8 + g;
      if (row >= D.rows) continue;
      double* drow = D.p + (long long)row * D.ld;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int col = j0 + wn * 32 + c * 8 + q * 2;
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

template <int NS, int NT, int STAGES>
static cudaError_t launch_cfg(const BatchArgs<double>& a, cudaStream_t s) {
  using namespace f64cfg;
  const size_t smem = (size_t)STAGES * (NS + NT) * BK * LDS * sizeof(double);
  auto kern = prod_f64_kernel<NS, NT, STAGES>;
  static bool attr_set = false;  // per-instantiation; benign race (idempotent)
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  kern<<<a.total_tiles, THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_batch_f64(const BatchArgs<double>& a, cudaStream_t s) {
  if (a.total_tiles <= 0) return cudaSuccess;
  int ns = 1, nt = 1;
  for (int i = 0; i < a.count; ++i) {
    ns = max(ns, a.p[i].ns);
    if (a.p[i].kind != kSyrk) nt = max(nt, a.p[i].nt);
  }
  if (ns == 1 && nt == 1) return launch_cfg<1, 1, 4>(a, s);
  if (ns == 2 && nt == 1) return launch_cfg<2, 1, 3>(a, s);
  if (ns == 1 && nt == 2) return launch_cfg<1, 2, 3>(a, s);
  return launch_cfg<2, 2, 3>(a, s);
}

int tile_rows_f64() { return f64cfg::BM; }

}  // namespace ata
