// Multi-node Strassen additions (sm_100a): one launch runs the combo4 (operand
// sums) or postadd7 (post-additions) passes of many independent nodes of one
// recursion level -- the breadth-first executions of reference-threshold
// recursions (ref_bfs.py) have thousands of small nodes per level, where one
// launch per node would be launch-latency bound.
//
// Node descriptors are compact windows packed into the kernel parameters
// (<= 30 KB per launch); blockIdx.z selects the node, blockIdx.x and the
// threads cover its rows x column-pairs as one flat range, with the same per-element arithmetic as the single-node
// kernels in elementwise.cu (zero-extended sources, truncated outputs).
#include <cstring>

#include "ata_common.cuh"

namespace ata {

namespace {

constexpr int kMtThreads = 256;

// Two adjacent elements (c0 even) with one 16-byte (f64) / 8-byte (f32) access
// when the window allows it: base aligned to two elements and an even pitch.
template <typename T> struct Pair;
template <> struct Pair<double> { using V = double2; };
template <> struct Pair<float> { using V = float2; };
template <typename T>
__device__ __forceinline__ bool pair_ok(const T* p, long long ld) {
  return ((reinterpret_cast<uintptr_t>(p) & (2 * sizeof(T) - 1)) == 0) && ((ld & 1) == 0);
}
template <typename T>
__device__ __forceinline__ void load_pair(const T* q, int avail, bool vec, T& x, T& y) {
  if (vec && avail >= 2) {
    const typename Pair<T>::V v = __ldcs(reinterpret_cast<const typename Pair<T>::V*>(q));
    x = v.x;
    y = v.y;
  } else {
    x = avail > 0 ? __ldcs(q) : T(0);
    y = avail > 1 ? __ldcs(q + 1) : T(0);
  }
}
template <typename T>
__device__ __forceinline__ void store_pair(T* q, int avail, bool vec, T x, T y, bool accumulate) {
  if (vec && avail >= 2) {
    typename Pair<T>::V* pv = reinterpret_cast<typename Pair<T>::V*>(q);
    if (accumulate) {
      const typename Pair<T>::V o = *pv;
      x += o.x;
      y += o.y;
    }
    typename Pair<T>::V v;
    v.x = x;
    v.y = y;
    *pv = v;
  } else {
    if (avail > 0) q[0] = accumulate ? q[0] + x : x;
    if (avail > 1) q[1] = accumulate ? q[1] + y : y;
  }
}

template <typename T>
struct Win {
  T* p;
  long long ld;
  int rows, cols;
};

template <typename T>
struct C4Node {
  Win<T> src[4];
  Win<T> dst[5];
  int code[5];
  int nsrc, ndst, rows, cols, lower;
};

template <typename T>
struct P7Node {
  Win<T> src[7];
  Win<T> dst[4];
  T sign[4];
  int rows, cols, accumulate, _pad;
};

constexpr int kC4Max = 104;
constexpr int kP7Max = 96;

template <typename T>
struct C4Batch {
  int count, maxrows;
  C4Node<T> n[kC4Max];
};
template <typename T>
struct P7Batch {
  int count, maxrows;
  P7Node<T> n[kP7Max];
};
static_assert(sizeof(C4Batch<double>) <= 30000 && sizeof(P7Batch<double>) <= 30000, "kernel parameter space");

// Work split: blockIdx.z = node; the node's rows x ceil(cols/2) column pairs
// are one flat index space over blockIdx.x and the 256 threads (consecutive
// threads take consecutive pairs of a row: coalesced), so narrow nodes of deep
// recursion levels keep every thread busy.
template <typename T>
__global__ void combo4_multi_kernel(const __grid_constant__ C4Batch<T> b) {
  const C4Node<T>& a = b.n[blockIdx.z];
  const int cp = (a.cols + 1) >> 1;
  const int x0 = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  const int dr = stride / cp, dc = stride - dr * cp;   // the flat index advanced incrementally
  int r = x0 / cp, cc = x0 - (x0 / cp) * cp;
  for (; r < a.rows; r += dr, cc += dc) {
    if (cc >= cp) {
      cc -= cp;
      if (++r >= a.rows) break;
    }
    const int c0 = cc * 2;
    T v[4][2];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[q][0] = v[q][1] = T(0);
      if (q < a.nsrc) {
        const Win<T>& S = a.src[q];
        const bool ok = r < S.rows;
        load_pair(S.p + (ok ? (long long)r * S.ld + c0 : 0), ok ? S.cols - c0 : 0, pair_ok(S.p, S.ld),
                  v[q][0], v[q][1]);
      }
    }
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      if (j >= a.ndst) break;
      const Win<T>& D = a.dst[j];
      if (r >= D.rows) continue;
      T o0 = T(0), o1 = T(0);
      int code = a.code[j];
#pragma unroll
      for (int q = 0; q < 4; ++q, code >>= 2) {
        const int cq = code & 3;
        if (cq == 1) o0 += v[q][0], o1 += v[q][1];
        else if (cq == 2) o0 -= v[q][0], o1 -= v[q][1];
      }
      const int cmax = a.lower ? min(D.cols, r + 1) : D.cols;
      store_pair(D.p + (long long)r * D.ld + c0, cmax - c0, pair_ok(D.p, D.ld), o0, o1, false);
    }
  }
}

template <typename T>
__global__ void postadd7_multi_kernel(const __grid_constant__ P7Batch<T> b) {
  const P7Node<T>& a = b.n[blockIdx.z];
  const int cp = (a.cols + 1) >> 1;
  const int x0 = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  const int dr = stride / cp, dc = stride - dr * cp;   // the flat index advanced incrementally
  int r = x0 / cp, cc = x0 - (x0 / cp) * cp;
  for (; r < a.rows; r += dr, cc += dc) {
    if (cc >= cp) {
      cc -= cp;
      if (++r >= a.rows) break;
    }
    const int c0 = cc * 2;
    T p[7][2];
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      const Win<T>& S = a.src[i];
      const bool ok = r < S.rows;
      load_pair(S.p + (ok ? (long long)r * S.ld + c0 : 0), ok ? S.cols - c0 : 0, pair_ok(S.p, S.ld),
                p[i][0], p[i][1]);
    }
    T o[4][2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      o[0][e] = p[0][e] + p[3][e] - p[4][e] + p[6][e];
      o[1][e] = p[2][e] + p[4][e];
      o[2][e] = p[1][e] + p[3][e];
      o[3][e] = p[0][e] - p[1][e] + p[2][e] + p[5][e];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const Win<T>& D = a.dst[j];
      if (r >= D.rows) continue;
      const T sg = a.sign[j];
      store_pair(D.p + (long long)r * D.ld + c0, D.cols - c0, pair_ok(D.p, D.ld), sg * o[j][0], sg * o[j][1],
                 a.accumulate != 0);
    }
  }
}

template <typename T>
Win<T> win_of(const DTerm<T>& t) {
  Win<T> w;
  w.p = const_cast<T*>(t.p);
  w.ld = t.ld;
  w.rows = t.rows;
  w.cols = t.cols;
  return w;
}
template <typename T>
Win<T> win_of(const DDest<T>& d) {
  Win<T> w;
  w.p = d.p;
  w.ld = d.ld;
  w.rows = d.rows;
  w.cols = d.cols;
  return w;
}

// grid for `count` nodes of at most maxcols x maxrows: ~32 blocks per SM in total
static dim3 multi_grid(int count, int maxrows, int maxcols) {
  // one block row per 256 column pairs of the largest node, capped so the
  // launch has ~16 blocks per SM (grid-stride loop inside)
  const long long pairs = (long long)maxrows * ((maxcols + 1) / 2);
  long long gx = (pairs + kMtThreads - 1) / kMtThreads;
#ifndef EWM_BLOCKS_PER_SM
#define EWM_BLOCKS_PER_SM 64  // measured on c2: 16 -> 64 blocks per SM per launch, 5.66 -> 5.27 ms
#endif
  const long long cap = 148LL * EWM_BLOCKS_PER_SM / count;
  if (gx > cap) gx = cap;
  if (gx < 1) gx = 1;
  return dim3((unsigned)gx, 1, count);
}

}  // namespace

template <typename T>
cudaError_t launch_combo4_multi(const EwArgs<T>* nodes, int count, cudaStream_t s) {
  for (int i = 0; i < count;) {
    C4Batch<T> b;
    std::memset(&b, 0, sizeof(b));
    int maxcols = 0;
    for (; i < count && b.count < kC4Max; ++i) {
      const EwArgs<T>& a = nodes[i];
      if (a.ndst > 5 || a.rows <= 0 || a.cols <= 0) {
        if (a.ndst > 5) return cudaErrorInvalidValue;  // the caller batches <= 5 outputs only
        continue;
      }
      C4Node<T>& n = b.n[b.count++];
      for (int q = 0; q < a.nsrc; ++q) n.src[q] = win_of(a.src[q]);
      for (int j = 0; j < a.ndst; ++j) {
        n.dst[j] = win_of(a.dst[j]);
        n.code[j] = a.dst[j].coef;
      }
      n.nsrc = a.nsrc;
      n.ndst = a.ndst;
      n.rows = a.rows;
      n.cols = a.cols;
      n.lower = a.lower;
      b.maxrows = b.maxrows > a.rows ? b.maxrows : a.rows;
      maxcols = maxcols > a.cols ? maxcols : a.cols;
    }
    if (b.count == 0) continue;
    combo4_multi_kernel<T><<<multi_grid(b.count, b.maxrows, maxcols), kMtThreads, 0, s>>>(b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <typename T>
cudaError_t launch_postadd7_multi(const EwArgs<T>* nodes, const int* accumulate, int count, cudaStream_t s) {
  for (int i = 0; i < count;) {
    P7Batch<T> b;
    std::memset(&b, 0, sizeof(b));
    int maxcols = 0;
    for (; i < count && b.count < kP7Max; ++i) {
      const EwArgs<T>& a = nodes[i];
      if (a.rows <= 0 || a.cols <= 0) continue;
      P7Node<T>& n = b.n[b.count++];
      for (int q = 0; q < 7; ++q) n.src[q] = win_of(a.src[q]);
      for (int j = 0; j < 4; ++j) {
        n.dst[j] = win_of(a.dst[j]);
        n.sign[j] = T(a.dst[j].sign);
      }
      n.rows = a.rows;
      n.cols = a.cols;
      n.accumulate = accumulate[i];
      b.maxrows = b.maxrows > a.rows ? b.maxrows : a.rows;
      maxcols = maxcols > a.cols ? maxcols : a.cols;
    }
    if (b.count == 0) continue;
    postadd7_multi_kernel<T><<<multi_grid(b.count, b.maxrows, maxcols), kMtThreads, 0, s>>>(b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template cudaError_t launch_combo4_multi<double>(const EwArgs<double>*, int, cudaStream_t);
template cudaError_t launch_combo4_multi<float>(const EwArgs<float>*, int, cudaStream_t);
template cudaError_t launch_postadd7_multi<double>(const EwArgs<double>*, const int*, int, cudaStream_t);
template cudaError_t launch_postadd7_multi<float>(const EwArgs<float>*, const int*, int, cudaStream_t);

}  // namespace ata
