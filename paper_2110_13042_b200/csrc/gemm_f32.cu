// FP32-storage generalized-product kernel, TF32 tensor-core multiply
// (mma.sync m16n8k8 tf32, fp32 accumulate).  Same product semantics as
// gemm_f64.cu (fused zero-extended operand terms, fused truncated
// destinations, SYRK lower-tile enumeration); see that file for the
// reference call sites it replaces.  This is the general-shape f32 path; the
// tall-skinny SYRK of config c5 goes through the tcgen05 kernel
// (syrk_tf32_tc.cu) when its shape allows.
#include <cstdlib>

#include "ata_common.cuh"

namespace ata {

namespace f32cfg {
constexpr int BM = 128, BN = 128, BK = 32, LDS = BM + 8, THREADS = 256;
}

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <bool VEC16>
__device__ __forceinline__ void load_term_f32(float* buf, const DTerm<float>& t, int l0, int c0,
                                              int tid) {
  using namespace f32cfg;
  if (VEC16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = (tid >> 5) + 8 * i;
      const int c = (tid & 31) * 4;
      const int gl = l0 + r, gc = c0 + c;
      int bytes = 0;
      if (gl < t.rows) {
        const int left = t.cols - gc;
        bytes = left >= 4 ? 16 : (left > 0 ? left * 4 : 0);
      }
      const float* src = bytes ? t.p + (long long)gl * t.ld + gc : t.p;
      cp_async_16(buf + r * LDS + c, src, bytes);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int r = (tid >> 7) + 2 * i;
      const int c = tid & 127;
      const int gl = l0 + r, gc = c0 + c;
      const int bytes = (gl < t.rows && gc < t.cols) ? 4 : 0;
      const float* src = bytes ? t.p + (long long)gl * t.ld + gc : t.p;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(buf + r * LDS + c)),
                   "l"(src), "r"(bytes));
    }
  }
}

template <bool VEC16>
__device__ __forceinline__ void combine_f32(float* buf0, const float* buf1, float sign1, int tid) {
  using namespace f32cfg;
  if (VEC16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = (tid >> 5) + 8 * i;
      const int c = (tid & 31) * 4;
      float4* x = reinterpret_cast<float4*>(buf0 + r * LDS + c);
      const float4 y = *reinterpret_cast<const float4*>(buf1 + r * LDS + c);
      float4 v = *x;
      v.x = fmaf(sign1, y.x, v.x);
      v.y = fmaf(sign1, y.y, v.y);
      v.z = fmaf(sign1, y.z, v.z);
      v.w = fmaf(sign1, y.w, v.w);
      *x = v;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int r = (tid >> 7) + 2 * i;
      const int c = tid & 127;
      buf0[r * LDS + c] = fmaf(sign1, buf1[r * LDS + c], buf0[r * LDS + c]);
    }
  }
}

__device__ __forceinline__ bool term_vec16_f32(const DTerm<float>& t) {
  return ((reinterpret_cast<uintptr_t>(t.p) & 15) == 0) && ((t.ld & 3) == 0);
}

// SPLIT = 3xTF32: x = hi + lo with hi = tf32(x), lo = tf32(x - hi); the
// product keeps hi*hi + hi*lo + lo*hi (fp32-level accuracy, 3 MMAs).  Without
// SPLIT a single TF32 MMA (config c5's TF32 leaves).
template <int NS, int NT, int STAGES, bool SPLIT>
__global__ void __launch_bounds__(f32cfg::THREADS, 1)
    prod_f32_kernel(const __grid_constant__ BatchArgs<float> args) {
  using namespace f32cfg;
  extern __shared__ __align__(128) float smemf[];
  constexpr int BUF = BK * LDS;
  constexpr int STAGE = (NS + NT) * BUF;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;

  const int tile = blockIdx.x;
  int pi = 0;
  while (pi + 1 < args.count && tile >= args.p[pi + 1].tile_begin) ++pi;
  const DProd<float>& P = args.p[pi];
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
  const int ns = P.ns, nt = syrk ? 1 : P.nt;
  const DTerm<float>& S0 = P.s[0];
  const DTerm<float>& S1 = P.s[1];
  const DTerm<float>& T0 = syrk ? P.s[0] : P.t[0];
  const DTerm<float>& T1 = P.t[1];
  const bool vs = term_vec16_f32(S0) && (ns < 2 || term_vec16_f32(S1));
  const bool vt = term_vec16_f32(T0) && (nt < 2 || term_vec16_f32(T1));

  auto load_stage = [&](int stage, int kt) {
    float* base = smemf + stage * STAGE;
    const int l0 = kt * BK;
    if (vs) load_term_f32<true>(base, S0, l0, i0, tid);
    else load_term_f32<false>(base, S0, l0, i0, tid);
    if (NS == 2 && ns == 2) {
      if (vs) load_term_f32<true>(base + BUF, S1, l0, i0, tid);
      else load_term_f32<false>(base + BUF, S1, l0, i0, tid);
    }
    float* tb = base + NS * BUF;
    if (vt) load_term_f32<true>(tb, T0, l0, j0, tid);
    else load_term_f32<false>(tb, T0, l0, j0, tid);
    if (NT == 2 && nt == 2) {
      if (vt) load_term_f32<true>(tb + BUF, T1, l0, j0, tid);
      else load_term_f32<false>(tb + BUF, T1, l0, j0, tid);
    }
  };

  // The tensor core's fp32 accumulation drops low-order bits (a negative bias
  // ~ additions x 2^-25 on sums of positive terms: -2.3e-4 on a 2^20-row Gram
  // diagonal, tools/acc_bias.py).  `acc` therefore only spans FLUSH k-tiles and
  // is added into `tot` on the CUDA cores (fp32, round to nearest).
  constexpr int FLUSH = SPLIT ? 1 : 8;
  float acc[4][4][4], tot[4][4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][b][e] = tot[a][b][e] = 0.f;

  const int KT = (P.m + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    const int stage = kt % STAGES;
    cp_async_wait<STAGES - 2>();
    float* base = smemf + stage * STAGE;
    if (NS == 2 && ns == 2) {
      if (vs) combine_f32<true>(base, base + BUF, (float)S1.sign, tid);
      else combine_f32<false>(base, base + BUF, (float)S1.sign, tid);
    }
    if (NT == 2 && nt == 2) {
      float* tb = base + NS * BUF;
      if (vt) combine_f32<true>(tb, tb + BUF, (float)T1.sign, tid);
      else combine_f32<false>(tb, tb + BUF, (float)T1.sign, tid);
    }
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT) load_stage(nk % STAGES, nk);
      cp_async_commit();
    }
    const float* As = base;
    const float* Bs = base + NS * BUF;
#pragma unroll
    for (int kk = 0; kk < BK / 8; ++kk) {
      uint32_t a[4][4], b[4][2], al[4][4], bl[4][2];
      const int r0 = (kk * 8 + q) * LDS, r1 = (kk * 8 + q + 4) * LDS;
      auto split = [&](float x, uint32_t& hi, uint32_t& lo) {
        hi = to_tf32(x);
        if (SPLIT) lo = to_tf32(x - __uint_as_float(hi));
      };
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int col = wm * 64 + mt * 16 + g;
        split(As[r0 + col], a[mt][0], al[mt][0]);
        split(As[r0 + col + 8], a[mt][1], al[mt][1]);
        split(As[r1 + col], a[mt][2], al[mt][2]);
        split(As[r1 + col + 8], a[mt][3], al[mt][3]);
      }
#pragma unroll
      for (int nt2 = 0; nt2 < 4; ++nt2) {
        const int col = wn * 32 + nt2 * 8 + g;
        split(Bs[r0 + col], b[nt2][0], bl[nt2][0]);
        split(Bs[r1 + col], b[nt2][1], bl[nt2][1]);
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt2 = 0; nt2 < 4; ++nt2) {
          if (SPLIT) {
            mma_tf32(acc[mt][nt2], al[mt], b[nt2]);
            mma_tf32(acc[mt][nt2], a[mt], bl[nt2]);
          }
          mma_tf32(acc[mt][nt2], a[mt], b[nt2]);
        }
    }
    if ((kt + 1) % FLUSH == 0 || kt == KT - 1) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            tot[a][b][e] += acc[a][b][e];
            acc[a][b][e] = 0.f;
          }
    }
  }
  cp_async_wait<0>();

  const int nd = P.nd;
  for (int d = 0; d < nd; ++d) {
    const DDest<float>& D = P.d[d];
    const float scale = (float)(args.alpha * D.sign);
    const bool accumulate = P.accumulate != 0;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = i0 + wm * 64 + mt * 16 + g + h * 8;
        if (row >= D.rows) continue;
        float* drow = D.p + (long long)row * D.ld;
#pragma unroll
        for (int nt2 = 0; nt2 < 4; ++nt2) {
          const int col = j0 + wn * 32 + nt2 * 8 + q * 2;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cc = col + e;
            if (cc < D.cols && (!syrk || cc <= row)) {
              const float v = scale * tot[mt][nt2][h * 2 + e];
              drow[cc] = accumulate ? drow[cc] + v : v;
            }
          }
        }
      }
    }
  }
}

template <int NS, int NT, int STAGES, bool SPLIT>
static cudaError_t launch_cfg_f32(const BatchArgs<float>& a, cudaStream_t s) {
  using namespace f32cfg;
  const size_t smem = (size_t)STAGES * (NS + NT) * BK * LDS * sizeof(float);
  auto kern = prod_f32_kernel<NS, NT, STAGES, SPLIT>;
  static std::atomic<unsigned long long> attr_set{0};
  if (cudaError_t e = ata::set_smem_attr(kern, smem, attr_set); e != cudaSuccess) return e;
  kern<<<a.total_tiles, THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

template <bool SPLIT>
static cudaError_t launch_batch_f32_t(BatchArgs<float> a, cudaStream_t s) {
  long long total = 0;
  for (int i = 0; i < a.count; ++i) {
    DProd<float>& p = a.p[i];
    p.tn = (p.n + f32cfg::BM - 1) / f32cfg::BM;
    p.tk = (p.k + f32cfg::BN - 1) / f32cfg::BN;
    p.tile_begin = (int)total;
    total += p.kind == kSyrk ? (long long)p.tn * (p.tn + 1) / 2 : (long long)p.tn * p.tk;
  }
  if (total <= 0) return cudaSuccess;
  if (total > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  a.total_tiles = (int)total;
  int ns = 1, nt = 1;
  for (int i = 0; i < a.count; ++i) {
    ns = max(ns, a.p[i].ns);
    if (a.p[i].kind != kSyrk) nt = max(nt, a.p[i].nt);
  }
  if (ns == 1 && nt == 1) return launch_cfg_f32<1, 1, 4, SPLIT>(a, s);
  if (ns == 2 && nt == 1) return launch_cfg_f32<2, 1, 3, SPLIT>(a, s);
  if (ns == 1 && nt == 2) return launch_cfg_f32<1, 2, 3, SPLIT>(a, s);
  return launch_cfg_f32<2, 2, 3, SPLIT>(a, s);
}

bool tc_eligible(const DProd<float>& p);
cudaError_t launch_tf32_tc(const DProd<float>* prods, int count, double alpha, cudaStream_t s);
cudaError_t launch_tf32_2sm(const DProd<float>* prods, int count, double alpha, cudaStream_t s);

cudaError_t launch_batch_f32(const BatchArgs<float>& a, cudaStream_t s, bool split) {
  if (split) return launch_batch_f32_t<true>(a, s);
  // single-pass TF32: plain products go to the tcgen05/TMA kernel, the rest
  // (fused multi-term / multi-destination products) to the mma.sync kernel
  static int use_tc = -1;
  if (use_tc < 0) {
    const char* e = std::getenv("ATA_TF32_TC");
    use_tc = e ? std::atoi(e) : 2;   // CTA pair by default (measured faster on c5 with KSUB flushes)
  }
  if (!use_tc) return launch_batch_f32_t<false>(a, s);
  DProd<float> tcp[kMaxBatch];
  int ntc = 0;
  BatchArgs<float> rest = a;
  rest.count = 0;
  for (int i = 0; i < a.count; ++i) {
    if (tc_eligible(a.p[i])) tcp[ntc++] = a.p[i];
    else rest.p[rest.count++] = a.p[i];
  }
  if (ntc > 0) {
    // 2 = CTA-pair tcgen05 kernel (cta_group::2), 1 = single-CTA tcgen05 kernel
    // (which has no L2 rounding ring: raw operands would be truncated -- refuse)
    if (use_tc != 2 && tf32_ring_pending()) return cudaErrorNotSupported;
    cudaError_t e = use_tc == 2 ? launch_tf32_2sm(tcp, ntc, a.alpha, s) : launch_tf32_tc(tcp, ntc, a.alpha, s);
    if (e != cudaSuccess) return e;
  }
  if (rest.count > 0) return launch_batch_f32_t<false>(rest, s);
  return cudaSuccess;
}


}  // namespace ata
