// Shared device-side descriptors and helpers for the AtA kernels (sm_100a).
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

namespace ata {

constexpr int kMaxBatch = 48;  // products per grouped launch (kernel-param by value, < 32 KB)
constexpr int kMaxDests = 8;  // destinations per product (ATA_MAX_DESTS)

template <typename T>
struct DTerm {  // zero-extended read window
  const T* p;
  long long ld;
  int rows, cols;
  double sign;
};

template <typename T>
struct DDest {  // truncated write window
  T* p;
  long long ld;
  int rows, cols;
  double sign;
  int sem;     // >= 0: base of this region's per-tile turn counters (ordered accumulation)
  int sem_ld;  // tile columns of the region (counter row pitch)
  int turn;    // this product's position in the region's accumulation order
  int coef;    // COMBO4 outputs: base-4 coefficient code over the sources
};

enum : int { kGemm = 0, kSyrk = 1 };

template <typename T, int MAXD>
struct DProdT {
  int kind;        // kGemm / kSyrk
  int m, n, k;     // contraction, output rows, output cols
  int ns, nt, nd;  // term / dest counts
  int accumulate;  // 1: D += v ; 0: D = v
  int tn, tk;      // tile grid (rows x cols); SYRK uses the lower triangle of tn x tn
  int tile_begin;  // prefix offset of this product in the launch's tile space
  int _pad;
  DTerm<T> s[2], t[2];
  DDest<T> d[MAXD];
};
template <typename T>
using DProd = DProdT<T, kMaxDests>;

template <typename T, int MAXD, int MAXB>
struct BatchArgsT {
  int count;
  int total_tiles;
  double alpha;
  int* sync;  // [0] = work counter, [1..] = destination turn counters (zeroed per launch)
  int n_sync;  // ints available at sync
  int dynamic; // 1: tiles handed out by the work counter (needed for ordered destinations)
  int dbg;     // experiment flags (ATA_DBG): 1 = skip ordering waits, 2 = skip epilogue
  DProdT<T, MAXD> p[MAXB];
};
template <typename T>
using BatchArgs = BatchArgsT<T, kMaxDests, kMaxBatch>;

// Narrow FP64 batches: products with <= 2 destinations (every planner's leaves)
// fit 104 to a launch (28 KB of parameters) instead of 48 -- groups of many
// small leaf products then give each persistent CTA several tiles.
constexpr int kNarrowDests = 2;
constexpr int kMaxBatchNarrow = 104;
using BatchArgsNarrow64 = BatchArgsT<double, kNarrowDests, kMaxBatchNarrow>;

// Unbounded FP64 batches of region-free narrow products: descriptors live in
// device memory (uploaded once per distinct batch, cached by content), with a
// tile -> product table; one persistent launch runs thousands of small
// products (breadth-first reference plans) with every CTA pipelining across
// many tiles.
template <typename T, int MAXD>
struct BatchArgsG {
  int count;
  int total_tiles;
  double alpha;
  int* sync;
  int n_sync;
  int dynamic;
  int dbg;
  const DProdT<T, MAXD>* gp;   // device array [count]
  const int* tile_prod;        // device array [total_tiles]: product of each tile
};
using BatchArgsGlobal64 = BatchArgsG<double, kNarrowDests>;
constexpr int kMaxBatchGlobal = 1 << 20;

template <typename T>
struct EwArgs {  // elementwise op: rows x cols iteration space
  int rows, cols, nsrc, ndst;
  int lower;  // combo4: write only elements with col <= row of each output window
  int _pad;
  DTerm<T> src[8];
  DDest<T> dst[kMaxDests];
};

// ---- host launchers (defined in gemm_*.cu / elementwise.cu) ----
cudaError_t launch_batch_f64(const BatchArgs<double>& a, cudaStream_t s);
cudaError_t launch_batch_f64_ws(const BatchArgs<double>& a, cudaStream_t s);
cudaError_t launch_batch_f64_narrow(const BatchArgsNarrow64& a, cudaStream_t s);
// count narrow region-free products with descriptors in host memory; returns
// cudaErrorNotReady when the descriptors are not resident and the stream is
// capturing a graph (the caller then launches them in narrow batches)
cudaError_t launch_batch_f64_global(DProdT<double, kNarrowDests>* prods, int count, double alpha, int* sync,
                                    cudaStream_t s);
bool f64_narrow_supported();
// single-term narrow products with TMA-legal windows (16-byte aligned, even
// pitch, cols % 16 == 0): one persistent launch of the TMA-fed kernel;
// cudaErrorNotReady while capturing with descriptors not yet resident
bool f64_tma_eligible(const DProdT<double, kNarrowDests>* prods, int count);
// `ride` (may be null): Strassen operand-sum nodes (combo4) of a LATER product
// group, independent of this launch's products, executed by the kernel's three
// spare producer warps per SM while the DMMAs run (f64_ride_eligible nodes only).
cudaError_t launch_batch_f64_tma(DProdT<double, kNarrowDests>* prods, int count, double alpha, int* sync,
                                 long long sync_ints, cudaStream_t s, const EwArgs<double>* ride = nullptr,
                                 int n_ride = 0);
bool f64_ride_eligible(const EwArgs<double>& node);
constexpr int kMaxRidePhases = 32;
bool f64_supports_ordering();
cudaError_t launch_batch_f32(const BatchArgs<float>& a, cudaStream_t s, bool split);
template <typename T> cudaError_t launch_combo(const EwArgs<T>& a, cudaStream_t s);
template <typename T> cudaError_t launch_update(const EwArgs<T>& a, cudaStream_t s);
template <typename T> cudaError_t launch_combo4(const EwArgs<T>& a, cudaStream_t s);
cudaError_t launch_round_tf32(const float* src, long long lds, float* dst, long long ldd, int rows, int cols,
                              cudaStream_t s);
// L2 rounding ring for the next single-pass TF32 product launch on this thread
// (ATA_OP_ROUND with accumulate == 2): the products read the raw rows of `a`;
// `buf` (buf_elems floats) holds the two rings and their flags.
struct Tf32Ring {
  const float* a;
  long long lda;
  int rows, cols;
  float* buf;
  long long buf_elems;
};
void set_tf32_ring(const Tf32Ring* r);  // nullptr clears
bool tf32_ring_pending();
template <typename T> cudaError_t launch_postadd7(const EwArgs<T>& a, int accumulate, cudaStream_t s);
// many independent nodes per launch (elementwise_multi.cu); combo4 nodes: <= 5 outputs
template <typename T> cudaError_t launch_combo4_multi(const EwArgs<T>* nodes, int count, cudaStream_t s);
template <typename T>
cudaError_t launch_postadd7_multi(const EwArgs<T>* nodes, const int* accumulate, int count, cudaStream_t s);
template <typename T> cudaError_t launch_fill(T* p, long long ld, int rows, int cols, cudaStream_t s);
template <typename T> cudaError_t launch_mirror(T* C, long long ldc, int n, cudaStream_t s);
template <typename T> cudaError_t launch_pack(const T* C, long long ldc, int n, T* packed, cudaStream_t s);
template <typename T>
cudaError_t launch_unpack(const T* packed, int n, T* C, long long ldc, int acc, cudaStream_t s);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async with zero-fill: copies src_bytes (0 or full) and zero-fills the rest.
__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_16(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Persistent grid size for a static round-robin tile schedule.  When the
// launch's products repeat with a period of P tiles (a contraction split into
// row chunks, each chunk = the same products over new rows) and P fits the
// machine, use a multiple of P workers so every wave runs whole chunks: the
// tiles sharing a chunk's operand panels then stream them in lockstep and the
// panels are read from HBM once (a chunk split across waves is read twice).
inline int periodic_workers(const int* tiles, const int* kinds, int n, long long total, int slots) {
  if (total <= slots) return (int)total;
  for (int q = 1; q <= n / 2; ++q) {
    if (n % q != 0) continue;
    bool same = true;
    for (int i = q; i < n && same; ++i) same = tiles[i] == tiles[i - q] && kinds[i] == kinds[i - q];
    if (!same) continue;
    long long period = 0;
    for (int i = 0; i < q; ++i) period += tiles[i];
    if (period > slots) break;
    const long long w = (slots / period) * period;
    return w * 10 >= (long long)slots * 9 ? (int)w : slots;
  }
  return slots;
}

// Host-side launch helpers.  The SM count and a kernel's max-dynamic-shared-
// memory attribute belong to a device (context), so both are cached per device
// ordinal: a process that drives several GPUs gets the attribute set on each.
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

inline int sm_count() {
  static std::atomic<int> cache[64];
  const int d = current_device();
  int n = (d >= 0 && d < 64) ? cache[d].load(std::memory_order_relaxed) : 0;
  if (n > 0) return n;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
  if (n <= 0) n = 148;
  if (d >= 0 && d < 64) cache[d].store(n, std::memory_order_relaxed);
  return n;
}

// `done` is one bit per device ordinal, owned by the caller (one static per
// kernel instantiation); setting the attribute twice is harmless.
template <typename Kernel>
inline cudaError_t set_smem_attr(Kernel kern, size_t smem, std::atomic<unsigned long long>& done) {
  const int d = current_device();
  const unsigned long long bit = (d >= 0 && d < 64) ? (1ull << d) : 0ull;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_release);
  return e;
}

}  // namespace ata
