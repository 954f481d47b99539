// C ABI + native plan executor (see include/atamul_b200.h).
//
// The executor walks a flat op list produced by the host planner, validates
// every window against its base buffer (a workspace overrun is the
// reference's WorkspaceUndersizedError, strassen.py:82-85), resolves windows
// into device pointers, coalesces consecutive same-group products into one
// grouped launch, and issues everything on one stream.  It never allocates and
// never synchronises, so a whole plan can be captured in a CUDA graph.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <type_traits>
#include <vector>

#include "../../include/atamul_b200.h"
#include "ata_common.cuh"

// kernel launches issued through the executor (reported by ata_launch_count)
static std::atomic<long long> g_launches{0};
// product launches that carried riding operand sums (reported by ata_ride_count)
static std::atomic<long long> g_rides{0};

namespace {

thread_local std::string g_last_error;



int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return ATA_E_CUDA;
}

struct Bases {
  const char* ptr[4];
  long long elems[4];
  size_t esize;
};

// Validate a window against its base. rows==0 or cols==0 means "empty/absent".
int check_ref(const ata_ref& r, const Bases& b, const char* what, int opi, bool write) {
  if (r.base < 0 || r.base > 3) return fail(ATA_E_ARG, std::string(what) + ": bad base");
  if (r.rows < 0 || r.cols < 0 || r.off < 0)
    return fail(ATA_E_SHAPE, "shape mismatch: negative window in op " + std::to_string(opi));
  if (r.rows == 0 || r.cols == 0) return ATA_OK;
  if (b.ptr[r.base] == nullptr)
    return fail(ATA_E_ARG, std::string(what) + ": null base pointer in op " + std::to_string(opi));
  if (r.rows > 1 && r.ld < r.cols)
    return fail(ATA_E_SHAPE, "shape mismatch: ld < cols in op " + std::to_string(opi));
  if (write && r.base == ATA_BASE_A)
    return fail(ATA_E_ARG, "op " + std::to_string(opi) + " writes into A");
  const long long last = r.off + (long long)(r.rows - 1) * r.ld + r.cols;
  if (last > b.elems[r.base]) {
    if (r.base == ATA_BASE_WS)
      return fail(ATA_E_WORKSPACE, "workspace undersized: op " + std::to_string(opi) + " needs " +
                                       std::to_string(last) + " scalars, have " +
                                       std::to_string(b.elems[r.base]));
    return fail(ATA_E_SHAPE, "shape mismatch: window exceeds its base buffer in op " +
                                 std::to_string(opi));
  }
  return ATA_OK;
}

template <typename T>
ata::DTerm<T> term_of(const ata_ref& r, const Bases& b) {
  ata::DTerm<T> t;
  t.p = reinterpret_cast<const T*>(b.ptr[r.base] ? b.ptr[r.base] + r.off * (long long)sizeof(T) : nullptr);
  t.ld = r.ld;
  t.rows = r.rows;
  t.cols = r.cols;
  t.sign = r.sign;
  if (t.p == nullptr) t.rows = t.cols = 0;
  return t;
}

template <typename T>
ata::DDest<T> dest_of(const ata_ref& r, const Bases& b) {
  ata::DDest<T> d;
  d.p = reinterpret_cast<T*>(const_cast<char*>(b.ptr[r.base]) + r.off * (long long)sizeof(T));
  d.ld = r.ld;
  d.rows = r.rows;
  d.cols = r.cols;
  d.sign = r.sign;
  return d;
}

template <typename T>
cudaError_t launch_batch(const ata::BatchArgs<T>& a, cudaStream_t s, int dtype);
template <>
cudaError_t launch_batch<double>(const ata::BatchArgs<double>& a, cudaStream_t s, int) {
  return ata::launch_batch_f64(a, s);
}
template <>
cudaError_t launch_batch<float>(const ata::BatchArgs<float>& a, cudaStream_t s, int dtype) {
  return ata::launch_batch_f32(a, s, dtype != ATA_TF32);
}

int validate_op(const ata_op& op, const Bases& b, int i) {
  int rc;
  if (op.ns < 0 || op.ns > ATA_MAX_TERMS || op.nt < 0 || op.nt > ATA_MAX_TERMS || op.nd < 0 ||
      op.nd > ATA_MAX_DESTS)
    return fail(ATA_E_ARG, "bad term/dest count in op " + std::to_string(i));
  for (int j = 0; j < op.ns; ++j)
    if ((rc = check_ref(op.s[j], b, "s", i, false))) return rc;
  for (int j = 0; j < op.nt; ++j)
    if ((rc = check_ref(op.t[j], b, "t", i, false))) return rc;
  for (int j = 0; j < op.nd; ++j)
    if ((rc = check_ref(op.d[j], b, "d", i, true))) return rc;
  switch (op.type) {
    case ATA_OP_GEMM:
    case ATA_OP_SYRK:
      if (op.m < 1 || op.n < 1 || op.k < 1 || op.ns < 1 || op.nd < 1 ||
          (op.type == ATA_OP_GEMM && op.nt < 1))
        return fail(ATA_E_SHAPE, "shape mismatch: empty product in op " + std::to_string(i));
      if (op.ns > 2 || op.nt > 2)
        return fail(ATA_E_ARG, "products take at most two terms per operand (op " + std::to_string(i) + ")");
      if (op.s[0].sign != 1.0 || (op.type == ATA_OP_GEMM && op.t[0].sign != 1.0))
        return fail(ATA_E_ARG, "leading operand term must have sign +1 (op " + std::to_string(i) + ")");
      for (int j = 0; j < op.ns; ++j)
        if (op.s[j].rows > op.m || op.s[j].cols > op.n)
          return fail(ATA_E_SHAPE, "shape mismatch: S term exceeds product in op " + std::to_string(i));
      for (int j = 0; j < op.nt; ++j)
        if (op.t[j].rows > op.m || op.t[j].cols > op.k)
          return fail(ATA_E_SHAPE, "shape mismatch: T term exceeds product in op " + std::to_string(i));
      for (int j = 0; j < op.nd; ++j)
        if (op.d[j].rows > op.n || op.d[j].cols > op.k)
          return fail(ATA_E_SHAPE, "shape mismatch: destination exceeds product in op " + std::to_string(i));
      if (op.type == ATA_OP_SYRK && op.n != op.k)
        return fail(ATA_E_SHAPE, "shape mismatch: SYRK output must be square");
      return ATA_OK;
    case ATA_OP_COMBO:
      if (op.nd != 1 || op.ns < 1) return fail(ATA_E_ARG, "combo needs 1 dest and >=1 term");
      for (int j = 0; j < op.ns; ++j)
        if (op.s[j].rows > op.d[0].rows + 1 || op.s[j].cols > op.d[0].cols + 1 ||
            op.s[j].rows < op.d[0].rows - 1 || op.s[j].cols < op.d[0].cols - 1)
          return fail(ATA_E_SHAPE, "shape mismatch: combo term differs by more than one row/col");
      return ATA_OK;
    case ATA_OP_UPDATE:
      if (op.ns != 1 || op.nd < 1) return fail(ATA_E_ARG, "update needs 1 source and >=1 dest");
      for (int j = 0; j < op.nd; ++j)
        if (op.d[j].rows > op.s[0].rows || op.d[j].cols > op.s[0].cols)
          return fail(ATA_E_SHAPE, "shape mismatch: update destination window exceeds source");
      return ATA_OK;
    case ATA_OP_FILL:
      if (op.nd != 1) return fail(ATA_E_ARG, "fill needs 1 dest");
      return ATA_OK;
    case ATA_OP_ROUND:
      if (op.accumulate == 2) {   // L2 ring: d[0] is the ring scratch (any shape), s[0] the raw operand
        if (op.ns != 1 || op.nd != 1) return fail(ATA_E_ARG, "ring round needs one source and one scratch window");
        if (b.esize != 4) return fail(ATA_E_ARG, "round: fp32 plans only");
        return ATA_OK;
      }
      if (op.ns != 1 || op.nd != 1 || op.s[0].rows != op.d[0].rows || op.s[0].cols != op.d[0].cols)
        return fail(ATA_E_SHAPE, "shape mismatch: round needs one source and one equal-shape dest");
      if (b.esize != 4) return fail(ATA_E_ARG, "round: fp32 plans only");
      return ATA_OK;
    case ATA_OP_POSTADD7:
      if (op.ns != 4 || op.nt != 3 || op.nd != 4)
        return fail(ATA_E_ARG, "postadd7 needs 7 children (s[0..3], t[0..2]) and 4 outputs");
      {
        int maxr = 0, maxc = 0;
        for (int q = 0; q < 7; ++q) {
          const ata_ref& c = q < 4 ? op.s[q] : op.t[q - 4];
          maxr = std::max(maxr, c.rows);
          maxc = std::max(maxc, c.cols);
        }
        for (int j = 0; j < 4; ++j)
          if (op.d[j].rows > maxr || op.d[j].cols > maxc)
            return fail(ATA_E_SHAPE, "shape mismatch: postadd7 output exceeds its children");
      }
      return ATA_OK;
    case ATA_OP_COMBO4:
      if (op.ns < 1 || op.nd < 1) return fail(ATA_E_ARG, "combo4 needs sources and dests");
      for (int j = 0; j < op.nd; ++j) {
        int code = op.d[j].region;
        if (code < 0 || code >= (1 << (2 * op.ns)))
          return fail(ATA_E_ARG, "combo4: bad coefficient code in op " + std::to_string(i));
        for (int q = 0; q < op.ns; ++q, code >>= 2)
          if ((code & 3) == 3) return fail(ATA_E_ARG, "combo4: bad coefficient digit");
      }
      return ATA_OK;
    default:
      return fail(ATA_E_ARG, "unknown op type " + std::to_string(op.type));
  }
}

template <typename T>
bool supports_ordering();
template <>
bool supports_ordering<double>() { return ata::f64_supports_ordering(); }
template <>
bool supports_ordering<float>() { return false; }

// Walk the op list with the executor's batching rule, calling on_batch(first, last)
// for every product launch [first, last), on_ew_run(first, last) for every run of
// COMBO4 / POSTADD7 ops sharing a group >= 0 (one multi-node launch) and on_ew(i)
// for every other elementwise op.
// Consecutive GEMM/SYRK ops with equal group >= 0 share a launch (at most
// kMaxBatch); when the launcher cannot order shared destinations, a product
// whose region already occurs in the open batch starts a new launch.
// on_batch(first, last, cont): cont = the group continues in the next launch
// (the batch was cut at kMaxBatch products), so the two may run concurrently
// when neither orders shared destinations.
// on_ride(first, last): a run of COMBO4 ops flagged ATA_OPF_RIDE (independent of
// the product group that follows; they may execute inside its launch).
template <typename F1, typename F2, typename F3, typename F4>
int walk_batches(const ata_op* ops, int n_ops, bool ordering, bool narrow, F1 on_batch, F2 on_ew,
                 F3 on_ew_run, F4 on_ride) {
  int first = -1, group = -1, count = 0;
  bool all_narrow = true;  // every product of the open batch has <= kNarrowDests destinations
  std::vector<int> regions;
  auto has_region = [](const ata_op& op) {
    for (int j = 0; j < op.nd; ++j)
      if (op.d[j].region > 0) return true;
    return false;
  };
  auto flush = [&](int end, bool cont = false) -> int {
    int rc = ATA_OK;
    if (count > 0) rc = on_batch(first, end, cont);
    first = -1;
    count = 0;
    regions.clear();
    return rc;
  };
  for (int i = 0; i < n_ops; ++i) {
    const ata_op& op = ops[i];
    int rc;
    if (op.type == ATA_OP_GEMM || op.type == ATA_OP_SYRK) {
      const bool same = count > 0 && op.group >= 0 && op.group == group;
      // region-free narrow FP64 batches are unbounded (device-resident descriptors)
      const bool nar = narrow && all_narrow && op.nd <= ata::kNarrowDests;
      const int cap = (nar && regions.empty() && !has_region(op)) ? ata::kMaxBatchGlobal
                      : nar ? ata::kMaxBatchNarrow : ata::kMaxBatch;
      bool join = same && count < cap;
      bool conflict = false;
      if (join && !ordering) {
        for (int j = 0; j < op.nd && !conflict; ++j)
          if (op.d[j].region > 0)
            for (int r : regions)
              if (r == op.d[j].region) conflict = true;
        join = !conflict;
      }
      if (!join && (rc = flush(i, same && !conflict))) return rc;
      if (count == 0) {
        first = i;
        all_narrow = true;
      }
      all_narrow = all_narrow && op.nd <= ata::kNarrowDests;
      ++count;
      group = op.group;
      for (int j = 0; j < op.nd; ++j)
        if (op.d[j].region > 0) regions.push_back(op.d[j].region);
      if (op.group < 0 && (rc = flush(i + 1))) return rc;
      continue;
    }
    if ((rc = flush(i))) return rc;
    if (op.type == ATA_OP_COMBO4 && (op.flags & ATA_OPF_RIDE)) {
      int j = i + 1;
      while (j < n_ops && ops[j].type == ATA_OP_COMBO4 && (ops[j].flags & ATA_OPF_RIDE)) ++j;
      if ((rc = on_ride(i, j))) return rc;
      i = j - 1;
      continue;
    }
    if ((op.type == ATA_OP_COMBO4 || op.type == ATA_OP_POSTADD7) && op.group >= 0) {
      // consecutive combo4 / postadd7 ops of one group: independent nodes, one launch
      int j = i + 1;
      while (j < n_ops && ops[j].type == op.type && ops[j].group == op.group) ++j;
      if ((rc = on_ew_run(i, j))) return rc;
      i = j - 1;
      continue;
    }
    if ((rc = on_ew(i))) return rc;
  }
  return flush(n_ops);
}

// Turn counters one launch needs: 1 work counter + one per tile of each shared region.
int64_t batch_sync_ints(const ata_op* ops, int first, int last) {
  const int TILE = 128;
  std::vector<std::pair<int, std::pair<int, int>>> reg;  // region -> (tile rows, tile cols)
  int64_t total = 1;
  for (int i = first; i < last; ++i)
    for (int j = 0; j < ops[i].nd; ++j) {
      const int r = ops[i].d[j].region;
      if (r <= 0) continue;
      const int tn = (ops[i].n + TILE - 1) / TILE, tk = (ops[i].k + TILE - 1) / TILE;
      bool found = false;
      for (auto& e : reg)
        if (e.first == r) {
          e.second.first = std::max(e.second.first, tn);
          e.second.second = std::max(e.second.second, tk);
          found = true;
        }
      if (!found) reg.push_back({r, {tn, tk}});
    }
  for (auto& e : reg) total += (int64_t)e.second.first * e.second.second;
  return total;
}

// Auxiliary streams + events of the current device for concurrent product
// launches (created once; the first plan runs before any graph capture).
struct ForkJoin {
  static constexpr int K = 8;
  cudaStream_t aux[K];
  cudaEvent_t fork, done[K];
  bool ok = false;
  // one set per (device, calling stream): plans on different streams (other
  // host threads) never share fork/join events
  static ForkJoin& get(cudaStream_t s) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, ForkJoin> per_stream;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    auto it = per_stream.find({dev, s});
    if (it != per_stream.end()) return it->second;
    ForkJoin& f = per_stream[{dev, s}];
    bool ok = cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming) == cudaSuccess;
    for (int k = 0; k < K && ok; ++k)
      ok = cudaStreamCreateWithFlags(&f.aux[k], cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&f.done[k], cudaEventDisableTiming) == cudaSuccess;
    f.ok = ok;
    if (!ok) cudaGetLastError();  // fall back to one stream
    return f;
  }
};

template <typename T>
ata::EwArgs<T> combo4_args(const ata_op& op, const Bases& b) {
  ata::EwArgs<T> a;
  std::memset(&a, 0, sizeof(a));
  a.nsrc = op.ns;
  a.ndst = op.nd;
  a.lower = op.accumulate;  // COMBO4: accumulate field = lower-triangular outputs
  for (int j = 0; j < op.ns; ++j) a.src[j] = term_of<T>(op.s[j], b);
  for (int j = 0; j < op.nd; ++j) {
    a.dst[j] = dest_of<T>(op.d[j], b);
    a.dst[j].coef = op.d[j].region;
    a.rows = a.rows > op.d[j].rows ? a.rows : op.d[j].rows;
    a.cols = a.cols > op.d[j].cols ? a.cols : op.d[j].cols;
  }
  return a;
}

template <typename T>
ata::EwArgs<T> postadd7_args(const ata_op& op, const Bases& b) {
  ata::EwArgs<T> a;
  std::memset(&a, 0, sizeof(a));
  a.nsrc = 7;
  a.ndst = 4;
  for (int q = 0; q < 7; ++q) {
    a.src[q] = term_of<T>(q < 4 ? op.s[q] : op.t[q - 4], b);
    a.rows = a.rows > a.src[q].rows ? a.rows : a.src[q].rows;
    a.cols = a.cols > a.src[q].cols ? a.cols : a.src[q].cols;
  }
  for (int j = 0; j < 4; ++j) a.dst[j] = dest_of<T>(op.d[j], b);
  return a;
}

template <typename T>
int run_plan_t(const ata_op* ops, int n_ops, const Bases& b, int* sync, int64_t sync_ints,
               double alpha, cudaStream_t s, int dtype) {
  for (int i = 0; i < n_ops; ++i) {
    int rc = validate_op(ops[i], b, i);
    if (rc) return rc;
  }
  const bool ordering = supports_ordering<T>();
  ata::BatchArgs<T> batch;
  thread_local static ata::BatchArgsNarrow64 nbatch;  // 28 KB: not on the stack
  const bool narrow = std::is_same<T, double>::value && ata::f64_narrow_supported();
  auto fill_batch = [&](auto& batch, int first, int last) {
    batch.alpha = alpha;
    batch.sync = sync;
    batch.n_sync = (int)(sync_ints < 0x7fffffff ? sync_ints : 0x7fffffff);
    std::vector<int> ids;  // batch-local region numbering (1-based)
    for (int i = first; i < last; ++i) {
      const ata_op& op = ops[i];
      auto& p = batch.p[batch.count++];
      p.kind = op.type == ATA_OP_SYRK ? ata::kSyrk : ata::kGemm;
      p.m = op.m;
      p.n = op.n;
      p.k = op.k;
      p.ns = op.ns;
      p.nt = op.type == ATA_OP_SYRK ? 0 : op.nt;
      p.nd = op.nd;
      p.accumulate = op.accumulate;
      for (int j = 0; j < op.ns; ++j) p.s[j] = term_of<T>(op.s[j], b);
      for (int j = 0; j < p.nt; ++j) p.t[j] = term_of<T>(op.t[j], b);
      for (int j = 0; j < op.nd; ++j) {
        p.d[j] = dest_of<T>(op.d[j], b);
        p.d[j].sem = 0;
        if (ordering && op.d[j].region > 0) {
          int id = 0;
          for (size_t q = 0; q < ids.size(); ++q)
            if (ids[q] == op.d[j].region) id = (int)q + 1;
          if (id == 0) {
            ids.push_back(op.d[j].region);
            id = (int)ids.size();
          }
          p.d[j].sem = id;
        }
      }
    }
  };
  // riding operand sums waiting for the next product launch: ops [ride_first, ride_last)
  int ride_first = 0, ride_last = 0;
  static const bool ride_enabled = [] {
    const char* e = std::getenv("ATA_RIDE");
    return e == nullptr || std::atoi(e) != 0;
  }();
  std::function<int(int, int)> run_ew_range;   // ops [first, last) as ordinary elementwise launches
  auto flush_ride = [&]() -> int {             // pending sums that cannot ride: ordinary launches, now
    if (ride_last <= ride_first) return ATA_OK;
    const int f = ride_first, l = ride_last;
    ride_first = ride_last = 0;
    return run_ew_range(f, l);
  };
  auto launch_one = [&](int first, int last, cudaStream_t ls) -> int {
    cudaStream_t s = ls;
    const int64_t need = batch_sync_ints(ops, first, last);
    if (ordering && need > 1 && (sync == nullptr || need > sync_ints))
      return fail(ATA_E_WORKSPACE, "workspace undersized: sync buffer needs " +
                                       std::to_string(need) + " ints, have " +
                                       std::to_string(sync_ints));
    bool nb = narrow;
    for (int i = first; i < last && nb; ++i) nb = ops[i].nd <= ata::kNarrowDests;
    if (!nb && last - first > ata::kMaxBatch) return fail(ATA_E_ARG, "internal: oversized product batch");
    if (nb) {
      if constexpr (std::is_same<T, double>::value) {
        {
          // single-term products with TMA-legal windows: the TMA-fed kernel, one
          // persistent launch (descriptors and tensor maps in device memory)
          struct {
            int count;
            double alpha;
            int* sync;
            int n_sync;
            ata::DProdT<double, ata::kNarrowDests>* p;
          } tb;
          std::vector<ata::DProdT<double, ata::kNarrowDests>> prods(last - first);
          std::memset(prods.data(), 0, sizeof(prods[0]) * prods.size());
          tb.count = 0;
          tb.p = prods.data();
          fill_batch(tb, first, last);
          if (ata::f64_tma_eligible(prods.data(), tb.count)) {
            cudaError_t e = cudaErrorNotSupported;
            if (ride_last > ride_first && ride_enabled) {
              // the launch carries the pending operand sums on its spare warps
              std::vector<ata::EwArgs<double>> ride;
              for (int i = ride_first; i < ride_last; ++i) ride.push_back(combo4_args<double>(ops[i], b));
              // (on a copy: the launcher rewrites the descriptors' region fields, and a
              // refused ride falls through to the plain launch below)
              auto with_ride = prods;
              e = ata::launch_batch_f64_tma(with_ride.data(), tb.count, alpha, sync, sync_ints, s, ride.data(),
                                            (int)ride.size());
              if (e == cudaSuccess) {
                ride_first = ride_last = 0;
                g_launches += 1;
                g_rides += 1;
                return ATA_OK;
              }
              if (e != cudaErrorNotReady && e != cudaErrorNotSupported) return cuda_fail(e, "product launch (tma+ride)");
              cudaGetLastError();
            }
            if (int rc = flush_ride()) return rc;
            e = ata::launch_batch_f64_tma(prods.data(), tb.count, alpha, sync, sync_ints, s);
            if (e == cudaSuccess) {
              g_launches += 1;
              return ATA_OK;
            }
            if (e != cudaErrorNotReady && e != cudaErrorNotSupported) return cuda_fail(e, "product launch (tma)");
            cudaGetLastError();   // not resident while capturing / no map: the cp.async kernels below
          }
        }
        if (int rc = flush_ride()) return rc;
        static const bool no_global = std::getenv("ATA_NO_GLOBAL_BATCH") != nullptr;  // A/B knob
        if (last - first > ata::kMaxBatchNarrow && !no_global) {
          // unbounded region-free batch: device-resident descriptors, one launch
          struct {
            int count;
            double alpha;
            int* sync;
            int n_sync;
            ata::DProdT<double, ata::kNarrowDests>* p;
          } vb;
          std::vector<ata::DProdT<double, ata::kNarrowDests>> prods(last - first);
          std::memset(prods.data(), 0, sizeof(prods[0]) * prods.size());
          vb.count = 0;
          vb.p = prods.data();
          fill_batch(vb, first, last);
          cudaError_t e = ata::launch_batch_f64_global(prods.data(), vb.count, alpha, sync, s);
          g_launches += 1;
          if (e == cudaSuccess) return ATA_OK;
          if (e != cudaErrorNotReady) return cuda_fail(e, "product launch");
          // capturing a graph with descriptors not yet resident: narrow batches instead
          for (int c0 = first; c0 < last; c0 += ata::kMaxBatchNarrow) {
            std::memset(&nbatch, 0, sizeof(nbatch));
            fill_batch(nbatch, c0, std::min(last, c0 + ata::kMaxBatchNarrow));
            e = ata::launch_batch_f64_narrow(nbatch, s);
            g_launches += 1;
            if (e != cudaSuccess) return cuda_fail(e, "product launch");
          }
          return ATA_OK;
        }
        for (int c0 = first; c0 < last; c0 += ata::kMaxBatchNarrow) {
          std::memset(&nbatch, 0, sizeof(nbatch));
          fill_batch(nbatch, c0, std::min(last, c0 + ata::kMaxBatchNarrow));
          cudaError_t e = ata::launch_batch_f64_narrow(nbatch, s);
          g_launches += 1;
          if (e != cudaSuccess) return cuda_fail(e, "product launch");
        }
        return ATA_OK;
      }
    }
    if (int rc = flush_ride()) return rc;
    std::memset(&batch, 0, sizeof(batch));
    fill_batch(batch, first, last);
    cudaError_t e = launch_batch<T>(batch, s, dtype);
    g_launches += 1;
    if (e != cudaSuccess) return cuda_fail(e, "product launch");
    return ATA_OK;
  };
  // Launches of one product group cut at kMaxBatch are independent: unless they
  // order shared destinations (turn counters in the sync buffer), they run
  // concurrently on auxiliary streams forked from / joined back into `s`, so
  // groups of many small products fill the machine (graph-capturable).
  ForkJoin& fj = ForkJoin::get(s);
  bool prev_cont = false;
  int aux_next = 0;
  bool forked = false, aux_used[ForkJoin::K] = {false};
  auto join_all = [&]() -> int {
    if (!forked) return ATA_OK;
    for (int k = 0; k < ForkJoin::K; ++k)
      if (aux_used[k]) {
        if (cudaEventRecord(fj.done[k], fj.aux[k]) != cudaSuccess ||
            cudaStreamWaitEvent(s, fj.done[k], 0) != cudaSuccess)
          return cuda_fail(cudaGetLastError(), "stream join");
        aux_used[k] = false;
      }
    forked = false;
    return ATA_OK;
  };
  auto on_batch = [&](int first, int last, bool cont) -> int {
    bool regions = false;
    for (int i = first; i < last && !regions; ++i)
      for (int j = 0; j < ops[i].nd; ++j) regions = regions || ops[i].d[j].region > 0;
    const bool concurrent = (cont || prev_cont) && !regions && fj.ok;
    if (!prev_cont || !concurrent) {  // a new group (or an ordered batch): serialise behind all prior work
      if (int rc = join_all()) return rc;
    }
    prev_cont = cont;
    cudaStream_t ls = s;
    if (concurrent) {
      if (!forked) {
        if (cudaEventRecord(fj.fork, s) != cudaSuccess) return cuda_fail(cudaGetLastError(), "stream fork");
        forked = true;
        aux_next = 0;
      }
      const int k = aux_next++ % ForkJoin::K;
      if (!aux_used[k]) {
        if (cudaStreamWaitEvent(fj.aux[k], fj.fork, 0) != cudaSuccess)
          return cuda_fail(cudaGetLastError(), "stream fork");
        aux_used[k] = true;
      }
      ls = fj.aux[k];
    }
    if (int rc = launch_one(first, last, ls)) return rc;
    if (!cont) return join_all();
    return ATA_OK;
  };
  auto on_ew = [&](int i) -> int {
    if (int rc = flush_ride()) return rc;
    if (int rc = join_all()) return rc;
    ata::set_tf32_ring(nullptr);   // a ring belongs to the product group right after its ROUND op
    g_launches += 1;
    const ata_op& op = ops[i];
    cudaError_t e = cudaSuccess;
    if (op.type == ATA_OP_COMBO || op.type == ATA_OP_UPDATE) {
      ata::EwArgs<T> a;
      std::memset(&a, 0, sizeof(a));
      a.nsrc = op.ns;
      a.ndst = op.nd;
      for (int j = 0; j < op.ns; ++j) a.src[j] = term_of<T>(op.s[j], b);
      for (int j = 0; j < op.nd; ++j) a.dst[j] = dest_of<T>(op.d[j], b);
      if (op.type == ATA_OP_COMBO) {
        a.rows = op.d[0].rows;
        a.cols = op.d[0].cols;
        e = ata::launch_combo<T>(a, s);
      } else {
        // iterate over the union of the destination windows (each <= source)
        for (int j = 0; j < op.nd; ++j) {
          a.rows = a.rows > op.d[j].rows ? a.rows : op.d[j].rows;
          a.cols = a.cols > op.d[j].cols ? a.cols : op.d[j].cols;
        }
        e = ata::launch_update<T>(a, s);
      }
    } else if (op.type == ATA_OP_FILL) {
      ata::DDest<T> d = dest_of<T>(op.d[0], b);
      e = ata::launch_fill<T>(d.p, d.ld, d.rows, d.cols, s);
    } else if (op.type == ATA_OP_COMBO4) {
      e = ata::launch_combo4<T>(combo4_args<T>(op, b), s);
    } else if (op.type == ATA_OP_ROUND && op.accumulate == 2) {
      // no pass: the next TF32 product group rounds its operands through the L2 ring
      const ata::DTerm<T> src = term_of<T>(op.s[0], b);
      const ata::DDest<T> dst = dest_of<T>(op.d[0], b);
      ata::Tf32Ring r;
      r.a = reinterpret_cast<const float*>(src.p);
      r.lda = src.ld;
      r.rows = src.rows;
      r.cols = src.cols;
      r.buf = reinterpret_cast<float*>(dst.p);
      r.buf_elems = (long long)dst.rows * dst.ld;
      ata::set_tf32_ring(&r);
      g_launches -= 1;
      return ATA_OK;
    } else if (op.type == ATA_OP_ROUND) {
      const ata::DTerm<T> src = term_of<T>(op.s[0], b);
      const ata::DDest<T> dst = dest_of<T>(op.d[0], b);
      e = ata::launch_round_tf32(reinterpret_cast<const float*>(src.p), src.ld, reinterpret_cast<float*>(dst.p),
                                 dst.ld, dst.rows, dst.cols, s);
    } else if (op.type == ATA_OP_POSTADD7) {
      e = ata::launch_postadd7<T>(postadd7_args<T>(op, b), op.accumulate, s);
    }
    if (e != cudaSuccess) return cuda_fail(e, "elementwise launch");
    return ATA_OK;
  };
  auto on_ew_run = [&](int first, int last) -> int {
    if (int rc = flush_ride()) return rc;
    if (int rc = join_all()) return rc;
    ata::set_tf32_ring(nullptr);
    std::vector<ata::EwArgs<T>> args;
    std::vector<int> acc;
    args.reserve(last - first);
    cudaError_t e = cudaSuccess;
    if (ops[first].type == ATA_OP_COMBO4) {
      bool small = true;
      for (int i = first; i < last; ++i) small = small && ops[i].nd <= 5;
      if (!small) {  // nodes with > 5 outputs: one launch each
        for (int i = first; i < last; ++i)
          if (int rc = on_ew(i)) return rc;
        return ATA_OK;
      }
      for (int i = first; i < last; ++i) args.push_back(combo4_args<T>(ops[i], b));
      e = ata::launch_combo4_multi<T>(args.data(), (int)args.size(), s);
      g_launches += (long long)(args.size() + 103) / 104;
    } else {
      for (int i = first; i < last; ++i) {
        args.push_back(postadd7_args<T>(ops[i], b));
        acc.push_back(ops[i].accumulate);
      }
      e = ata::launch_postadd7_multi<T>(args.data(), acc.data(), (int)args.size(), s);
      g_launches += (long long)(args.size() + 95) / 96;
    }
    if (e != cudaSuccess) return cuda_fail(e, "elementwise launch");
    return ATA_OK;
  };
  run_ew_range = [&](int first, int last) -> int {
    for (int i = first; i < last;) {
      int j = i + 1;
      if (ops[i].group >= 0) {
        while (j < last && ops[j].group == ops[i].group) ++j;
        if (int rc = on_ew_run(i, j)) return rc;
      } else if (int rc = on_ew(i)) {
        return rc;
      }
      i = j;
    }
    return ATA_OK;
  };
  auto on_ride = [&](int first, int last) -> int {
    if (int rc = flush_ride()) return rc;
    ride_first = first;
    ride_last = last;
    return ATA_OK;
  };
  int rc = walk_batches(ops, n_ops, ordering, narrow, on_batch, on_ew, on_ew_run, on_ride);
  if (rc == ATA_OK) rc = flush_ride();
  int rj = join_all();
  ata::set_tf32_ring(nullptr);
  return rc ? rc : rj;
}

}  // namespace

extern "C" {

const char* ata_last_error(void) { return g_last_error.c_str(); }

const char* ata_strerror(int code) {
  switch (code) {
    case ATA_OK: return "ok";
    case ATA_E_SHAPE: return "shape mismatch";
    case ATA_E_UNSPLITTABLE: return "unsplittable";
    case ATA_E_WORKSPACE: return "workspace undersized";
    case ATA_E_UNSUPPORTED: return "unsupported size";
    case ATA_E_PROTOCOL: return "protocol error";
    case ATA_E_CUDA: return "cuda error";
    case ATA_E_ARG: return "invalid argument";
    default: return "unknown error";
  }
}

int ata_version(void) { return 100; }
int64_t ata_launch_count(void) { return (int64_t)g_launches.load(); }
int64_t ata_ride_count(void) { return (int64_t)g_rides.load(); }
int ata_abi_op_size(void) { return (int)sizeof(ata_op); }

int64_t ata_sync_ints_needed(int dtype, const ata_op* ops, int32_t n_ops) {
  if (n_ops <= 0 || ops == nullptr) return 1;
  const bool ordering = dtype == ATA_F64 ? ata::f64_supports_ordering() : false;
  const bool narrow = dtype == ATA_F64 && ata::f64_narrow_supported();
  int64_t need = 1;
  bool rides = false;
  walk_batches(
      ops, n_ops, ordering, narrow,
      [&](int first, int last, bool) -> int {
        need = std::max(need, batch_sync_ints(ops, first, last));
        return ATA_OK;
      },
      [](int) -> int { return ATA_OK; }, [](int, int) -> int { return ATA_OK; },
      [&](int, int) -> int {
        rides = true;
        return ATA_OK;
      });
  // riding operand sums: a chunk queue and one count per phase behind the turn counters
  return need + (rides ? 1 + ata::kMaxRidePhases : 0);
}

int ata_run_plan(int dtype, const ata_op* ops, int32_t n_ops, const void* A, int64_t a_elems,
                 const void* B, int64_t b_elems, void* C, int64_t c_elems, void* WS,
                 int64_t ws_elems, void* sync, int64_t sync_ints, double alpha, void* stream) {
  if (n_ops < 0 || (n_ops > 0 && ops == nullptr)) return fail(ATA_E_ARG, "null op list");
  Bases b;
  b.ptr[ATA_BASE_A] = static_cast<const char*>(A);
  b.ptr[ATA_BASE_C] = static_cast<const char*>(C);
  b.ptr[ATA_BASE_WS] = static_cast<const char*>(WS);
  b.ptr[ATA_BASE_B] = static_cast<const char*>(B);
  b.elems[ATA_BASE_A] = a_elems;
  b.elems[ATA_BASE_C] = c_elems;
  b.elems[ATA_BASE_WS] = ws_elems;
  b.elems[ATA_BASE_B] = b_elems;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == ATA_F64) {
    b.esize = 8;
    return run_plan_t<double>(ops, n_ops, b, static_cast<int*>(sync), sync_ints, alpha, s, dtype);
  }
  if (dtype == ATA_F32 || dtype == ATA_TF32) {
    b.esize = 4;
    return run_plan_t<float>(ops, n_ops, b, static_cast<int*>(sync), sync_ints, alpha, s, dtype);
  }
  return fail(ATA_E_ARG, "unknown dtype");
}

static ata_ref mkref(int base, long long ld, int rows, int cols) {
  ata_ref r;
  std::memset(&r, 0, sizeof(r));
  r.base = base;
  r.off = 0;
  r.ld = ld;
  r.rows = rows;
  r.cols = cols;
  r.sign = 1.0;
  return r;
}

int ata_syrk_lower(int dtype, const void* A, int64_t lda, int32_t m, int32_t n, void* C,
                   int64_t ldc, double alpha, void* stream) {
  if (m < 1 || n < 1) return fail(ATA_E_SHAPE, "shape mismatch: empty operand");
  ata_op op;
  std::memset(&op, 0, sizeof(op));
  op.type = ATA_OP_SYRK;
  op.m = m;
  op.n = n;
  op.k = n;
  op.ns = 1;
  op.nd = 1;
  op.accumulate = 1;
  op.group = -1;
  op.s[0] = mkref(ATA_BASE_A, lda, m, n);
  op.d[0] = mkref(ATA_BASE_C, ldc, n, n);
  const long long ae = (long long)(m - 1) * lda + n, ce = (long long)(n - 1) * ldc + n;
  return ata_run_plan(dtype, &op, 1, A, ae, nullptr, 0, C, ce, nullptr, 0, nullptr, 0, alpha, stream);
}

int ata_gemm_atb(int dtype, const void* A, int64_t lda, const void* B, int64_t ldb, int32_t m,
                 int32_t n, int32_t k, void* C, int64_t ldc, double alpha, void* stream) {
  if (m < 1 || n < 1 || k < 1) return fail(ATA_E_SHAPE, "shape mismatch: empty operand");
  ata_op op;
  std::memset(&op, 0, sizeof(op));
  op.type = ATA_OP_GEMM;
  op.m = m;
  op.n = n;
  op.k = k;
  op.ns = 1;
  op.nt = 1;
  op.nd = 1;
  op.accumulate = 1;
  op.group = -1;
  op.s[0] = mkref(ATA_BASE_A, lda, m, n);
  op.t[0] = mkref(ATA_BASE_B, ldb, m, k);
  op.d[0] = mkref(ATA_BASE_C, ldc, n, k);
  const long long ae = (long long)(m - 1) * lda + n, be = (long long)(m - 1) * ldb + k,
                  ce = (long long)(n - 1) * ldc + k;
  return ata_run_plan(dtype, &op, 1, A, ae, B, be, C, ce, nullptr, 0, nullptr, 0, alpha, stream);
}

int ata_add_truncated(int dtype, void* dst, int64_t ldd, int32_t dr, int32_t dc, const void* src,
                      int64_t lds, int32_t sr, int32_t sc, double scale, void* stream) {
  if (dr < 1 || dc < 1 || sr < 1 || sc < 1) return fail(ATA_E_SHAPE, "shape mismatch: empty block");
  if (dr - sr > 1 || sr - dr > 1 || dc - sc > 1 || sc - dc > 1)
    return fail(ATA_E_SHAPE, "shape mismatch: add_truncated (" + std::to_string(dr) + "," +
                                 std::to_string(dc) + ") vs (" + std::to_string(sr) + "," +
                                 std::to_string(sc) + ")");
  const int r = dr < sr ? dr : sr, c = dc < sc ? dc : sc;
  ata_op op;
  std::memset(&op, 0, sizeof(op));
  op.type = ATA_OP_UPDATE;
  op.ns = 1;
  op.nd = 1;
  op.group = -1;
  op.s[0] = mkref(ATA_BASE_A, lds, sr, sc);
  op.d[0] = mkref(ATA_BASE_C, ldd, r, c);
  op.d[0].sign = scale;
  const long long se = (long long)(sr - 1) * lds + sc, de = (long long)(dr - 1) * ldd + dc;
  return ata_run_plan(dtype, &op, 1, src, se, nullptr, 0, dst, de, nullptr, 0, nullptr, 0, 1.0, stream);
}

int ata_mirror_lower(int dtype, void* C, int64_t ldc, int32_t n, void* stream) {
  if (n < 1 || C == nullptr) return fail(ATA_E_SHAPE, "shape mismatch: mirror needs a square block");
  cudaError_t e = dtype == ATA_F64
                      ? ata::launch_mirror<double>(static_cast<double*>(C), ldc, n, (cudaStream_t)stream)
                      : ata::launch_mirror<float>(static_cast<float*>(C), ldc, n, (cudaStream_t)stream);
  g_launches += 1;
  return e == cudaSuccess ? ATA_OK : cuda_fail(e, "mirror");
}

int ata_pack_lower(int dtype, const void* C, int64_t ldc, int32_t n, void* packed, void* stream) {
  if (n < 1 || C == nullptr || packed == nullptr) return fail(ATA_E_SHAPE, "shape mismatch: pack_lower");
  cudaError_t e =
      dtype == ATA_F64
          ? ata::launch_pack<double>(static_cast<const double*>(C), ldc, n, static_cast<double*>(packed),
                                     (cudaStream_t)stream)
          : ata::launch_pack<float>(static_cast<const float*>(C), ldc, n, static_cast<float*>(packed),
                                    (cudaStream_t)stream);
  g_launches += 1;
  return e == cudaSuccess ? ATA_OK : cuda_fail(e, "pack");
}

int ata_unpack_lower(int dtype, const void* packed, int32_t n, void* C, int64_t ldc,
                     int32_t accumulate, void* stream) {
  if (n < 1 || C == nullptr || packed == nullptr) return fail(ATA_E_SHAPE, "shape mismatch: unpack_lower target");
  cudaError_t e = dtype == ATA_F64
                      ? ata::launch_unpack<double>(static_cast<const double*>(packed), n,
                                                   static_cast<double*>(C), ldc, accumulate,
                                                   (cudaStream_t)stream)
                      : ata::launch_unpack<float>(static_cast<const float*>(packed), n,
                                                  static_cast<float*>(C), ldc, accumulate,
                                                  (cudaStream_t)stream);
  g_launches += 1;
  return e == cudaSuccess ? ATA_OK : cuda_fail(e, "unpack");
}

}  // extern "C"
