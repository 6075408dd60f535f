// Whole-matrix host-buffer entry point: the GPU replacement of MatrixJob.run over the
// compiled kernel module (pkg/src/pcflib/matrix.py:156-234: pack once, fill every row
// block, return the dense M x M array; _sweepkern.pack / fill_block, pyx:72-121).
//
// One call takes the reference's pack() layout in host memory (tcat, vcat, off) and
// returns the dense matrix in host memory, original order.  On the device:
//
//   H2D (SoA + size sort + plan) -> K3 pack -> diagonal -> K1/K1c/K1r/K1g fills over a
//   queue in column-sweep order, cut into cost-balanced CHUNKS  ==>  D2H of the rows each
//   chunk finishes on two copy streams while later chunks compute.
//
// Row s of the size-sorted order is complete once every item whose row block contains s
// (its pairs (s, q > s)) and every item whose columns contain s (row blocks before s) has
// run.  The queue sweeps the column ranges right to left, so the short high rows finish
// first and few rows remain at the end; the host computes, per chunk, the rows it
// finishes (the last chunk touching each row), and the D2H of those rows (one contiguous
// M-entry row per PCF, scattered through perm to its original row) overlaps the compute of
// the later chunks.  The 80 GB result of the 100k benchmark leaves the device while the
// kernel runs instead of after it.  With one kernel kind the whole queue is ONE
// persistent launch whose items bump per-chunk completion counters
// (cuStreamWaitValue32 on the copy streams).
//
// Device buffers come from a grow-only workspace kept between calls (like a caching
// allocator); pcf_release_workspace() frees it.
#include <dlfcn.h>
#include <stdio.h>
#include <sys/mman.h>
#include <stdlib.h>
#include <string.h>
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <memory>
#include <numeric>
#include <vector>
#include "pcf_internal.h"

namespace pcfb {
namespace {

int fail(cudaError_t e, const char* where) {
  set_error("%s: %s", where, cudaGetErrorString(e));
  return PCF_ERR_CUDA;
}

// grow-only device workspace, one slot per buffer role
enum Slot { W_T, W_V, W_OFF, W_PERM, W_SOFF, W_GOFF, W_RECS, W_RECSG, W_TILE, W_ITEMS, W_CNT,
            W_ERR, W_OUT, W_TAG, W_DONE, W_NSLOT };
struct Workspace {
  int device = -1;
  void* p[W_NSLOT] = {};
  size_t sz[W_NSLOT] = {};
  cudaStream_t s0 = nullptr, s1 = nullptr, s2 = nullptr;
  void release() {
    for (int k = 0; k < W_NSLOT; ++k) {
      if (p[k]) cudaFree(p[k]);
      p[k] = nullptr;
      sz[k] = 0;
    }
    if (s0) cudaStreamDestroy(s0);
    if (s1) cudaStreamDestroy(s1);
    if (s2) cudaStreamDestroy(s2);
    s0 = s1 = s2 = nullptr;
    device = -1;
  }
  cudaError_t get(Slot k, size_t bytes, void** out) {
    bytes = bytes ? bytes : 16;
    if (sz[k] < bytes) {
      if (p[k]) cudaFree(p[k]);
      p[k] = nullptr;
      sz[k] = 0;
      cudaError_t e = cudaMalloc(&p[k], bytes);
      if (e != cudaSuccess) return e;
      sz[k] = bytes;
    }
    *out = p[k];
    return cudaSuccess;
  }
};
Workspace g_ws;
std::mutex g_ws_mutex;  // one whole-matrix call at a time per process (shared workspace)

// row copy list for one chunk: original row perm[s] of the device matrix to the same row
// of the host matrix, for every sorted row s the chunk finishes
cudaError_t copy_rows(const std::vector<int32_t>& perm, const std::vector<int32_t>& rows,
                      const char* dsrc, char* hdst, int64_t M, int64_t ld, size_t es,
                      cudaStream_t st) {
  const size_t n = rows.size();
  static const bool no_d2h = getenv("PCF_HOST_NO_D2H") != nullptr;  // timing experiments
  if (n == 0 || no_d2h) return cudaSuccess;
  // original row indices in ascending order, coalesced into runs of consecutive rows:
  // one pitched copy per run (source pitch M, host pitch ld)
  std::vector<int64_t> o(n);
  for (size_t k = 0; k < n; ++k) o[k] = perm[rows[k]];
  std::sort(o.begin(), o.end());
  const size_t row_bytes = (size_t)M * es;
  for (size_t k = 0; k < n;) {
    size_t e = k + 1;
    while (e < n && o[e] == o[e - 1] + 1) ++e;
    char* h = hdst + (size_t)o[k] * (size_t)ld * es;
    const char* d = dsrc + (size_t)o[k] * row_bytes;
    // contiguous on both sides (one row, or ld == M): a plain 1-D copy
    const cudaError_t rc =
        (e - k == 1 || ld == M)
            ? cudaMemcpyAsync(h, d, row_bytes * (e - k), cudaMemcpyDeviceToHost, st)
            : cudaMemcpy2DAsync(h, (size_t)ld * es, d, row_bytes, row_bytes, e - k,
                                cudaMemcpyDeviceToHost, st);
    if (rc != cudaSuccess) return rc;
    k = e;
  }
  return cudaSuccess;
}

// ---- result in pageable host memory (e.g. the numpy array pdist returns): pinning an
// 80 GB result costs ~56 s on the GPU box (1.4 GB/s), so the finished rows go through a
// small pinned staging pool instead -- D2H into a slot, host worker threads copy the slot's
// rows to their places (transparent huge pages requested for the result), slot reused.
struct PinnedPool {
  char* p = nullptr;
  size_t bytes = 0;
  ~PinnedPool() {
    if (p) cudaFreeHost(p);
  }
  cudaError_t get(size_t n, char** out) {
    if (bytes < n) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      bytes = 0;
      cudaError_t e = cudaHostAlloc((void**)&p, n, cudaHostAllocDefault);
      if (e != cudaSuccess) return e;
      bytes = n;
    }
    *out = p;
    return cudaSuccess;
  }
};
PinnedPool g_pin;

class Stager {
 public:
  Stager(char* out, int64_t M, int64_t ld, size_t es, const char* d_out, char* pool, int nslot,
         size_t slot_rows)
      : out_(out), M_(M), ld_(ld), es_(es), d_out_(d_out), nslot_(nslot), slot_rows_(slot_rows) {
    const size_t row = (size_t)M * es;
    for (int k = 0; k < nslot; ++k) {
      slot_.push_back(pool + (size_t)k * slot_rows * row);
      cudaEvent_t ev = nullptr;
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      ev_.push_back(ev);
      free_.push_back(k);
    }
    const unsigned hw = std::thread::hardware_concurrency();
    int nw = (int)std::max(2u, std::min(16u, hw ? hw : 4u));
    if (const char* ev = getenv("PCF_STAGE_WORKERS")) nw = std::max(1, atoi(ev));
    for (int w = 0; w < nw; ++w) workers_.emplace_back([this] { work(); });
  }
  ~Stager() { finish(); }
  // D2H of the given original rows (ascending) on stream st, through the slots
  cudaError_t drain(const std::vector<int64_t>& rows, cudaStream_t st) {
    const size_t row = (size_t)M_ * es_;
    for (size_t k0 = 0; k0 < rows.size(); k0 += slot_rows_) {
      const size_t k1 = std::min(rows.size(), k0 + slot_rows_);
      int slot;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return !free_.empty() || err_; });
        if (err_) return cudaErrorUnknown;
        slot = free_.front();
        free_.pop_front();
      }
      for (size_t k = k0; k < k1;) {  // runs of consecutive rows: one copy each
        size_t e = k + 1;
        while (e < k1 && rows[e] == rows[e - 1] + 1) ++e;
        const cudaError_t rc =
            cudaMemcpyAsync(slot_[slot] + (k - k0) * row, d_out_ + (size_t)rows[k] * row,
                            row * (e - k), cudaMemcpyDeviceToHost, st);
        if (rc != cudaSuccess) return rc;
        k = e;
      }
      cudaError_t rc = cudaEventRecord(ev_[slot], st);
      if (rc != cudaSuccess) return rc;
      {
        std::lock_guard<std::mutex> lk(mu_);
        q_.push_back(Piece{slot, std::vector<int64_t>(rows.begin() + k0, rows.begin() + k1)});
      }
      cv_.notify_all();
    }
    return cudaSuccess;
  }
  // wait for every queued row to reach the result; returns false on a CUDA error
  bool finish() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      done_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
    workers_.clear();
    for (auto ev : ev_)
      if (ev) cudaEventDestroy(ev);
    ev_.clear();
    return !err_;
  }

 private:
  struct Piece {
    int slot;
    std::vector<int64_t> rows;
  };
  void work() {
    const size_t row = (size_t)M_ * es_;
    for (;;) {
      Piece pc;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return !q_.empty() || done_; });
        if (q_.empty()) return;
        pc = std::move(q_.front());
        q_.pop_front();
      }
      const bool ok = cudaEventSynchronize(ev_[pc.slot]) == cudaSuccess;
      if (ok)
        for (size_t k = 0; k < pc.rows.size(); ++k)
          memcpy(out_ + (size_t)pc.rows[k] * (size_t)ld_ * es_, slot_[pc.slot] + k * row, row);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (!ok) err_ = true;
        free_.push_back(pc.slot);
      }
      cv_.notify_all();
    }
  }
  char* out_;
  int64_t M_, ld_;
  size_t es_;
  const char* d_out_;
  int nslot_;
  size_t slot_rows_;
  std::vector<char*> slot_;
  std::vector<cudaEvent_t> ev_;
  std::deque<int> free_;
  std::deque<Piece> q_;
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_;
  bool done_ = false, err_ = false;
};

// cuStreamWaitValue32 from the driver (opened at run time; null if unavailable): lets the
// copy stream wait on the fill kernel's per-chunk completion counters, so the whole
// matrix runs as ONE persistent launch (no per-chunk launch tails)
typedef int (*WaitValue32)(void* stream, unsigned long long addr, unsigned int value,
                           unsigned int flags);
WaitValue32 stream_wait_fn() {
  static WaitValue32 fn = [] {
    if (getenv("PCF_NO_STREAM_WAIT")) return (WaitValue32) nullptr;
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_LOCAL);
    if (!h) return (WaitValue32) nullptr;
    void* f = dlsym(h, "cuStreamWaitValue32_v2");
    if (!f) f = dlsym(h, "cuStreamWaitValue32");
    return (WaitValue32)f;
  }();
  return fn;
}

}  // namespace
}  // namespace pcfb

using namespace pcfb;

extern "C" {

void pcf_release_workspace(void) {
  std::lock_guard<std::mutex> lock(g_ws_mutex);
  g_ws.release();
}

int pcf_matrix_host(const void* tcat, const void* vcat, int is_f32, const int64_t* off, int64_t M,
                    int op, double p, int apply_root, int diag, double a, double b,
                    int32_t max_log2G, int32_t n_chunks, void* out, int64_t ld, int64_t* err_i,
                    int64_t* err_j, void* stream) {
  if (err_i) *err_i = -1;
  if (err_j) *err_j = -1;
  if (!tcat || !vcat || !off || !out || M < 1 || ld < M || !pcf_op_ok(op) ||
      !(a >= 0.0) || !(a < b) || M > 0x7fffffff) {
    set_error("pcf_matrix_host: bad arguments");
    return PCF_ERR_ARG;
  }
  if (n_chunks < 1) n_chunks = 1;
  std::lock_guard<std::mutex> lock(g_ws_mutex);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(e, "pcf_matrix_host device");
  if (g_ws.device != dev) {
    g_ws.release();
    g_ws.device = dev;
  }
  if (!g_ws.s0) {
    if ((e = cudaStreamCreateWithFlags(&g_ws.s0, cudaStreamNonBlocking)) ||
        (e = cudaStreamCreateWithFlags(&g_ws.s1, cudaStreamNonBlocking)) ||
        (e = cudaStreamCreateWithFlags(&g_ws.s2, cudaStreamNonBlocking)))
      return fail(e, "pcf_matrix_host streams");
  }
  // compute on the caller's stream (events around the call then bracket all of its
  // device work), copies on a second stream joined back into it before returning
  cudaStream_t s0 = stream ? (cudaStream_t)stream : g_ws.s0, s1 = g_ws.s1, s2 = g_ws.s2;

  // ---- host: size sort (descending, stable), sorted offsets, group offsets, plan
  const bool timing = getenv("PCF_HOST_TIMING") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  auto ms_since = [&](std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
        .count();
  };
  const int64_t N = off[M] - off[0];
  std::vector<int64_t> sizes(M);
  for (int64_t i = 0; i < M; ++i) {
    sizes[i] = off[i + 1] - off[i];
    if (sizes[i] < 1) {
      set_error("pcf_matrix_host: PCF %lld has no rows", (long long)i);
      return PCF_ERR_ARG;
    }
  }
  // the raw time / value arrays go up first: their H2D overlaps the host planning below
  const size_t es = is_f32 ? 4 : 8;
  void *d_t, *d_v;
  if ((e = g_ws.get(W_T, N * es, &d_t)) || (e = g_ws.get(W_V, N * es, &d_v)))
    return fail(e, "pcf_matrix_host alloc");
  // PCF_HOST_TIMING: device-side phase marks on s0 (upload start, fill start/end, done)
  cudaEvent_t tev[4] = {nullptr, nullptr, nullptr, nullptr};
  if (timing)
    for (auto& ev : tev) cudaEventCreate(&ev);
  if (timing) cudaEventRecord(tev[0], s0);
  if ((e = cudaMemcpyAsync(d_t, (const char*)tcat + off[0] * es, N * es, cudaMemcpyHostToDevice,
                           s0)) ||
      (e = cudaMemcpyAsync(d_v, (const char*)vcat + off[0] * es, N * es, cudaMemcpyHostToDevice,
                           s0)))
    return fail(e, "pcf_matrix_host upload");
  std::vector<int32_t> perm(M);
  std::iota(perm.begin(), perm.end(), 0);
  std::stable_sort(perm.begin(), perm.end(),
                   [&](int32_t x, int32_t y) { return sizes[x] > sizes[y]; });
  std::vector<int64_t> ss(M), soff(M + 1, 0);
  for (int64_t s = 0; s < M; ++s) {
    ss[s] = sizes[perm[s]];
    soff[s + 1] = soff[s] + ss[s];
  }
  const int rec_bytes = is_f32 ? 8 : 16;
  const int GW = 128 / rec_bytes;
  std::vector<int64_t> goff((M + GW - 1) / GW + 1);
  // (errors from here on first wait for the uploads already reading the caller's buffers)
  int rc = pcf_group_offsets(ss.data(), M, GW, goff.data());
  if (rc) return cudaStreamSynchronize(s0), rc;
  const double sort_ms = ms_since(t_start);
  int64_t n_items = 0;
  int32_t smem = 0;
  static const int max_cols = getenv("PCF_HOST_MAX_COLS") ? atoi(getenv("PCF_HOST_MAX_COLS")) : 2048;
  // one planner pass into a generous buffer (App-A 100k: 2.5 items per PCF); a second
  // pass only if it was too small
  std::vector<pcf_work_item> items((size_t)std::max<int64_t>(1024, 4 * M));
  rc = pcf_plan_pairwise(ss.data(), M, kPlanSmemBudget, max_cols, max_log2G, rec_bytes, items.data(),
                         (int64_t)items.size(), &n_items, &smem);
  if (rc == PCF_ERR_ARG && n_items > (int64_t)items.size()) {
    items.resize((size_t)n_items);
    rc = pcf_plan_pairwise(ss.data(), M, kPlanSmemBudget, max_cols, max_log2G, rec_bytes,
                           items.data(), n_items, &n_items, &smem);
  }
  if (rc) return cudaStreamSynchronize(s0), rc;
  items.resize(n_items);
  const double plan_ms = ms_since(t_start);

  // ---- queue order: a right-to-left sweep over column ranges (col0 descending, then
  // longest first).  Output row s is final once every item touching it has run -- its own
  // row block's items and the items whose column range holds s -- and in sweep order the
  // high (short, cheap) rows finish first and only the first few columns' rows finish at
  // the end, so the D2H of the M x M result runs beside the fill instead of after it (row
  // order would release half of the 80 GB in the last ~15% of the fill).
  auto item_cells = [&](const pcf_work_item& w) {
    const double rows_pts = (double)(soff[w.row0 + w.nrows] - soff[w.row0]);
    return (double)w.nrows * (double)(soff[w.col1] - soff[w.col0]) +
           (double)(w.col1 - w.col0) * rows_pts;
  };
  static const bool row_order = getenv("PCF_HOST_ROW_ORDER") != nullptr;  // A/B timing
  // kernel-major (one persistent launch per kernel), then the sweep within each kernel
  auto mode_rank = [](int m) { return m == 1 ? 0 : (m == 3 ? 1 : (m == 4 ? 2 : (m == 2 ? 3 : 4))); };
  std::stable_sort(items.begin(), items.end(), [&](const pcf_work_item& x, const pcf_work_item& y) {
    const int mx = mode_rank(x.smem_mode), my = mode_rank(y.smem_mode);
    if (mx != my) return mx < my;
    if (row_order) return x.row0 < y.row0;
    if (x.col0 != y.col0) return x.col0 > y.col0;
    return x.cost_hi > y.cost_hi;
  });
  double total = 0.0;
  for (auto& w : items) total += item_cells(w);
  struct Chunk { int64_t i0, i1; };
  std::vector<Chunk> chunks;
  {
    const int64_t nc = std::max<int64_t>(n_chunks, 512);
    int64_t start = 0;
    double acc = 0.0;
    for (int64_t i = 0; i < n_items; ++i) {
      acc += item_cells(items[i]);
      if (acc >= total / nc || i + 1 == n_items) {
        chunks.push_back({start, i + 1});
        start = i + 1;
        acc = 0.0;
      }
    }
    if (chunks.empty()) chunks.push_back({0, 0});
  }
  // rows finished by each chunk: done[s] = the last chunk touching s (assigned from the
  // last chunk down, each row once, via a next-unassigned skip list)
  std::vector<std::vector<int32_t>> chunk_rows(chunks.size());
  {
    std::vector<int32_t> owner(M, -1);
    std::vector<int64_t> nxt(M + 1);
    std::iota(nxt.begin(), nxt.end(), 0);
    auto find = [&](int64_t x) {
      int64_t r = x;
      while (nxt[r] != r) r = nxt[r];
      while (nxt[x] != r) {
        const int64_t t = nxt[x];
        nxt[x] = r;
        x = t;
      }
      return r;
    };
    auto claim = [&](int64_t lo, int64_t hi, int32_t k) {
      for (int64_t x = find(lo); x < hi; x = find(x)) {
        owner[x] = k;
        nxt[x] = x + 1;
      }
    };
    for (int64_t k = (int64_t)chunks.size() - 1; k >= 0; --k)
      for (int64_t i = chunks[k].i0; i < chunks[k].i1; ++i) {
        const pcf_work_item& w = items[i];
        claim(w.row0, std::min<int64_t>(w.row0 + w.nrows, M), (int32_t)k);
        claim(std::max<int64_t>(w.col0, w.row0 + 1), w.col1, (int32_t)k);
      }
    for (int64_t x = 0; x < M; ++x) chunk_rows[owner[x] < 0 ? 0 : owner[x]].push_back((int32_t)x);
  }
  // inside a chunk: one run per kernel (K1, K1c, K1s, K1r, K1g), each longest-first
  for (auto& ch : chunks) {
    std::stable_sort(items.begin() + ch.i0, items.begin() + ch.i1,
                     [&](const pcf_work_item& x, const pcf_work_item& y) {
                       const int mx = mode_rank(x.smem_mode), my = mode_rank(y.smem_mode);
                       if (mx != my) return mx < my;
                       return x.cost_hi > y.cost_hi;
                     });
  }

  const double host_ms = ms_since(t_start);
  // ---- device buffers
  void *d_off, *d_perm, *d_soff, *d_goff, *d_recs, *d_recsg, *d_tile, *d_items,
      *d_cnt, *d_err, *d_out;
  const int64_t ng = goff.back();
  if ((e = g_ws.get(W_OFF, (M + 1) * 8, &d_off)) || (e = g_ws.get(W_PERM, M * 4, &d_perm)) ||
      (e = g_ws.get(W_SOFF, (M + 1) * 8, &d_soff)) ||
      (e = g_ws.get(W_GOFF, goff.size() * 8, &d_goff)) ||
      (e = g_ws.get(W_RECS, N * 16, &d_recs)) ||
      (e = g_ws.get(W_RECSG, ng * (size_t)rec_bytes, &d_recsg)) ||
      (e = g_ws.get(W_TILE, is_f32 ? (N + 2) * 8 : 16, &d_tile)) ||
      (e = g_ws.get(W_ITEMS, std::max<int64_t>(n_items, 1) * sizeof(pcf_work_item), &d_items)) ||
      (e = g_ws.get(W_CNT, 64, &d_cnt)) || (e = g_ws.get(W_ERR, 8, &d_err)) ||
      (e = g_ws.get(W_OUT, (size_t)M * (size_t)M * es, &d_out)))
    return cudaStreamSynchronize(s0), fail(e, "pcf_matrix_host alloc");

  // rebase offsets to 0 if the caller passed a slice
  std::vector<int64_t> off0;
  const int64_t* offp = off;
  if (off[0] != 0) {
    off0.resize(M + 1);
    for (int64_t i = 0; i <= M; ++i) off0[i] = off[i] - off[0];
    offp = off0.data();
  }
  if ((e = cudaMemcpyAsync(d_off, offp, (M + 1) * 8, cudaMemcpyHostToDevice, s0)) ||
      (e = cudaMemcpyAsync(d_perm, perm.data(), M * 4, cudaMemcpyHostToDevice, s0)) ||
      (e = cudaMemcpyAsync(d_soff, soff.data(), (M + 1) * 8, cudaMemcpyHostToDevice, s0)) ||
      (e = cudaMemcpyAsync(d_goff, goff.data(), goff.size() * 8, cudaMemcpyHostToDevice, s0)) ||
      (e = cudaMemcpyAsync(d_items, items.data(), n_items * sizeof(pcf_work_item),
                           cudaMemcpyHostToDevice, s0)) ||
      (e = cudaMemsetAsync(d_err, 0xff, 8, s0)))
    return fail(e, "pcf_matrix_host upload");
  // K3 pack (float64 records for the diagonal and K1r/K1g of float64; float32 collections
  // also get the 8-byte tile records)
  if (!is_f32) {
    e = launch_pack(d_t, d_v, 0, (const int64_t*)d_off, (const int32_t*)d_perm,
                    (const int64_t*)d_soff, M, d_recs, (const int64_t*)d_goff, d_recsg, s0);
  } else {
    e = launch_pack(d_t, d_v, 1, (const int64_t*)d_off, (const int32_t*)d_perm,
                    (const int64_t*)d_soff, M, d_recs, nullptr, nullptr, s0);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_tile, 0, (N + 2) * 8, s0);
    if (e == cudaSuccess)
      e = launch_pack32((const float*)d_t, (const float*)d_v, (const int64_t*)d_off,
                        (const int32_t*)d_perm, (const int64_t*)d_soff, M, d_tile,
                        (const int64_t*)d_goff, d_recsg, s0);
  }
  if (e) return fail(e, "pcf_matrix_host pack");
  if ((e = launch_diag(d_recs, (const int64_t*)d_soff, (const int32_t*)d_perm, M, diag, a, b, d_out,
                       is_f32, M, (unsigned long long*)d_err, s0)))
    return fail(e, "pcf_matrix_host diagonal");

  FillArgs A;
  A.recs = is_f32 ? d_tile : d_recs;
  A.recs8 = d_recsg;
  A.soff = (const int64_t*)d_soff;
  A.goff8 = (const int64_t*)d_goff;
  A.perm = (const int32_t*)d_perm;
  A.M = M;
  A.counter = (int*)d_cnt;
  A.op = op;
  A.p = p;
  A.a = a;
  A.b = b;
  A.apply_root = apply_root;
  A.out = d_out;
  A.out_f32 = is_f32;
  A.ld = M;
  A.err = (unsigned long long*)d_err;
  A.smem_bytes = smem;
  A.rec_bytes = rec_bytes;
  {
    int n = 0;
    A.num_sms = (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
                 n > 0) ? n : 148;
  }
  std::vector<cudaEvent_t> evs(chunks.size(), nullptr);
  int status = PCF_OK;
  // result in pinned memory: rows go straight to it; pageable: through the staging pool
  cudaPointerAttributes pattr;
  const bool pinned_out = cudaPointerGetAttributes(&pattr, out) == cudaSuccess &&
                          pattr.type == cudaMemoryTypeHost;
  cudaGetLastError();
  std::unique_ptr<Stager> stager;
  if (!pinned_out) {
    const size_t row = (size_t)M * es;
    // 16 x 64 MB slots, one host copy thread per core (<= 16): c3 drain after the fill
    // 133 -> 120 ms against 8 x 128 MB with hw / 2 threads (tools/time_stage.py)
    size_t slot_mb = 64;
    int nslot = 16;
    if (const char* ev = getenv("PCF_STAGE_MB")) slot_mb = std::max(1, atoi(ev));
    if (const char* ev = getenv("PCF_STAGE_SLOTS")) nslot = std::max(2, atoi(ev));
    const size_t slot_rows = std::max<size_t>(1, std::min<size_t>((size_t)M, (slot_mb << 20) / row));
    char* pool = nullptr;
    if ((e = g_pin.get((size_t)nslot * slot_rows * row, &pool)))
      return cudaStreamSynchronize(s0), fail(e, "pcf_matrix_host staging pool");
    {  // transparent huge pages for the result: 512x fewer first-touch page faults
      const uintptr_t b = ((uintptr_t)out + (2u << 20) - 1) & ~(uintptr_t)((2u << 20) - 1);
      const uintptr_t en = ((uintptr_t)out + (size_t)M * (size_t)ld * es) & ~(uintptr_t)((2u << 20) - 1);
      if (en > b) madvise((void*)b, en - b, MADV_HUGEPAGE);
    }
    stager.reset(new Stager((char*)out, M, ld, es, (const char*)d_out, pool, nslot, slot_rows));
  }
  auto drain = [&](size_t k, cudaStream_t sc) -> cudaError_t {
    if (!stager) return copy_rows(perm, chunk_rows[k], (const char*)d_out, (char*)out, M, ld, es, sc);
    std::vector<int64_t> o(chunk_rows[k].size());
    for (size_t x = 0; x < o.size(); ++x) o[x] = perm[chunk_rows[k][x]];
    std::sort(o.begin(), o.end());
    return stager->drain(o, sc);
  };
  const WaitValue32 wait = stream_wait_fn();
  bool single = false;
  if (n_items > 0 && wait) {
    // ONE persistent launch per kernel over its run of the queue (kernel-major order);
    // item i bumps done[chunk(i)]; the copy streams wait for each chunk's count, then
    // drain its rows
    std::vector<int32_t> tag(n_items);
    for (size_t k = 0; k < chunks.size(); ++k)
      for (int64_t i = chunks[k].i0; i < chunks[k].i1; ++i) tag[i] = (int32_t)k;
    void *d_tag, *d_done;
    cudaEvent_t zeroed = nullptr;
    if ((e = g_ws.get(W_TAG, n_items * 4, &d_tag)) ||
        (e = g_ws.get(W_DONE, chunks.size() * 4, &d_done)) ||
        (e = cudaMemcpyAsync(d_tag, tag.data(), n_items * 4, cudaMemcpyHostToDevice, s0)) ||
        (e = cudaMemsetAsync(d_done, 0, chunks.size() * 4, s0)) ||
        (e = cudaEventCreateWithFlags(&zeroed, cudaEventDisableTiming)) ||
        (e = cudaEventRecord(zeroed, s0)) || (e = cudaStreamWaitEvent(s1, zeroed, 0)) ||
        (e = cudaStreamWaitEvent(s2, zeroed, 0)))
      return fail(e, "pcf_matrix_host single-launch setup");
    evs[0] = zeroed;  // destroyed with the others
    A.tag_done = (int32_t*)d_done;
    if (timing) cudaEventRecord(tev[1], s0);
    for (int64_t i = 0; i < n_items;) {
      int64_t j = i;
      while (j < n_items && items[j].smem_mode == items[i].smem_mode) ++j;
      A.items = (const PcfWorkItem*)d_items + i;
      A.n_items = (int)(j - i);
      A.smem_mode = items[i].smem_mode;
      A.item_tag = (const int32_t*)d_tag + i;
      if ((e = cudaMemsetAsync(d_cnt, 0, 4, s0)) || (e = launch_fill_tiles(A, s0)))
        return fail(e, "pcf_matrix_host fill");
      i = j;
    }
    if (timing) cudaEventRecord(tev[2], s0);
    single = true;
    for (size_t k = 0; k < chunks.size() && status == PCF_OK; ++k) {
      // chunks alternate between two copy streams (more DMA in flight over PCIe); chunk
      // k's rows need every chunk <= k finished: this stream already waited for k - 2 and
      // k - 3, so it waits for k - 1 and k
      cudaStream_t sc = (k & 1) ? s2 : s1;
      for (size_t j = k > 0 ? k - 1 : 0; j <= k && status == PCF_OK; ++j) {
        const unsigned n_j = (unsigned)(chunks[j].i1 - chunks[j].i0);
        int r = wait((void*)sc, (unsigned long long)((int32_t*)d_done + j), n_j, 0 /*GEQ*/);
        if (r) {
          set_error("pcf_matrix_host: cuStreamWaitValue32 failed (%d)", r);
          status = PCF_ERR_CUDA;
        }
      }
      if (status) break;
      if ((e = drain(k, sc))) {
        status = fail(e, "pcf_matrix_host drain");
        break;
      }
    }
  }
  for (size_t k = 0; !single && k < chunks.size() && status == PCF_OK; ++k) {
    const Chunk& ch = chunks[k];
    for (int64_t i = ch.i0; i < ch.i1;) {
      int64_t j = i;
      while (j < ch.i1 && items[j].smem_mode == items[i].smem_mode) ++j;
      A.items = (const PcfWorkItem*)d_items + i;
      A.n_items = (int)(j - i);
      A.smem_mode = items[i].smem_mode;
      if ((e = cudaMemsetAsync(d_cnt, 0, 4, s0)) || (e = launch_fill_tiles(A, s0))) {
        status = fail(e, "pcf_matrix_host fill");
        break;
      }
      i = j;
    }
    if (status) break;
    if ((e = cudaEventCreateWithFlags(&evs[k], cudaEventDisableTiming)) ||
        (e = cudaEventRecord(evs[k], s0)) || (e = cudaStreamWaitEvent(s1, evs[k], 0)) ||
        (e = drain(k, s1))) {
      status = fail(e, "pcf_matrix_host drain");
      break;
    }
  }
  unsigned long long key = ~0ull;
  cudaEvent_t join = nullptr;
  if (status == PCF_OK) {
    if ((e = cudaEventCreateWithFlags(&join, cudaEventDisableTiming)) ||
        (e = cudaEventRecord(join, s1)) || (e = cudaStreamWaitEvent(s0, join, 0)) ||
        (e = cudaEventRecord(join, s2)) || (e = cudaStreamWaitEvent(s0, join, 0)) ||
        (e = cudaMemcpyAsync(&key, d_err, 8, cudaMemcpyDeviceToHost, s0)) ||
        (timing && (e = cudaEventRecord(tev[3], s0))) || (e = cudaStreamSynchronize(s0)))
      status = fail(e, "pcf_matrix_host sync");
    if (join) cudaEventDestroy(join);
  } else {
    cudaStreamSynchronize(s0);
    cudaStreamSynchronize(s1);
    cudaStreamSynchronize(s2);
  }
  if (stager && !stager->finish() && status == PCF_OK)
    status = fail(cudaErrorUnknown, "pcf_matrix_host staged drain");
  for (auto ev : evs)
    if (ev) cudaEventDestroy(ev);
  if (timing) {
    fprintf(stderr, "pcf_matrix_host: host prep %.1f ms (sort %.1f, plan %.1f, order %.1f), "
            "total %.1f ms, %zu chunks, %lld items\n", host_ms, sort_ms, plan_ms - sort_ms,
            host_ms - plan_ms, ms_since(t_start), chunks.size(), (long long)n_items);
    float up = 0.f, fill = 0.f, tail = 0.f;
    if (single && status == PCF_OK) {
      cudaEventElapsedTime(&up, tev[0], tev[1]);
      cudaEventElapsedTime(&fill, tev[1], tev[2]);
      cudaEventElapsedTime(&tail, tev[2], tev[3]);
      fprintf(stderr, "pcf_matrix_host: device: upload+pack+diag %.1f ms, fill %.1f ms, "
              "drain after fill %.1f ms\n", up, fill, tail);
    }
  }
  for (auto ev : tev)
    if (ev) cudaEventDestroy(ev);
  if (status) return status;
  if (key != ~0ull) {
    if (err_i) *err_i = (int64_t)(key / (unsigned long long)M);
    if (err_j) *err_j = (int64_t)(key % (unsigned long long)M);
  }
  return PCF_OK;
}

}  // extern "C"
