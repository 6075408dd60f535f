// Kernel-plugin handle: the reference's _Backend.pack / fill_block pair
// (pkg/src/pcflib/_backend.py:40-46 -> _sweepkern.pack / fill_block, pyx:72-121) on the
// B200 engine, for a ctypes plugin inside the reference.
//
// The reference calls pack() once per MatrixJob (matrix.py:169-171) and then fill_block on
// disjoint row blocks [r0, r1) from `workers` threads concurrently (matrix.py:173-227).
// Here pack() uploads the collection once and packs it size-sorted on the device
// (pcf_collection_create).  The first fill_block of a job computes the WHOLE matrix with the
// tile kernels (K1 / K1c / K1r / K1s / K1g over the planner's work queue, one persistent
// launch per kernel run) into a device-resident float64 matrix cached on the handle; every
// fill_block -- including that first one -- then copies its rows [r0, r1), j >= i (j > i
// without the diagonal), and their mirrored columns into the caller's host matrix.  The
// per-block contract of fill_block is kept exactly: the first non-finite entry of the block
// in row-major order is returned as (i, j) and the entries after it stay untouched
// (pyx:104-121).  Entries are computed in float64 and rounded to the output kind on the
// host copy, as the reference stores <floating>acc (pyx:115-116).
//
// Default plan: exact (one lane per pair, the reference's left-to-right sum, libm pow),
// so fill_block == integrate_pair bit for bit as in the reference
// (tests/test_matrix.py:41-47); max_log2G > 0 selects the fast plan.
#include <math.h>
#include <sys/mman.h>
#include <stdlib.h>
#include <string.h>
#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <vector>
#include "pcf_internal.h"

namespace pcfb {
namespace {

int pfail(cudaError_t e, const char* where) {
  set_error("%s: %s", where, cudaGetErrorString(e));
  return PCF_ERR_CUDA;
}

struct MatKey {
  int op, apply_root, diag, lg;
  double p, a, b;
  bool operator==(const MatKey& o) const {
    return op == o.op && apply_root == o.apply_root && diag == o.diag && lg == o.lg &&
           memcmp(&p, &o.p, 8) == 0 && memcmp(&a, &o.a, 8) == 0 && memcmp(&b, &o.b, 8) == 0;
  }
};

struct Matrix {  // a computed M x M float64 matrix (original order) on the device
  MatKey key;
  double* d = nullptr;
  ~Matrix() {
    if (d) cudaFree(d);
  }
};

struct Plan {
  std::vector<pcf_work_item> items;
  pcf_work_item* d_items = nullptr;
  int32_t smem = 0;
};

struct Collection {
  int device = 0;
  int64_t M = 0, N = 0;
  int is_f32 = 0;
  std::vector<int32_t> perm;
  std::vector<int64_t> ss, soff, goff;
  void *d_perm = nullptr, *d_soff = nullptr, *d_goff = nullptr, *d_recs = nullptr,
       *d_recsg = nullptr, *d_tile = nullptr, *d_err = nullptr, *d_cnt = nullptr;
  cudaStream_t st = nullptr;
  std::mutex mu;
  std::map<int, Plan> plans;
  std::shared_ptr<Matrix> mat;
  ~Collection() {
    for (auto& kv : plans)
      if (kv.second.d_items) cudaFree(kv.second.d_items);
    for (void* q : {d_perm, d_soff, d_goff, d_recs, d_recsg, d_tile, d_err, d_cnt})
      if (q) cudaFree(q);
    if (st) cudaStreamDestroy(st);
  }
};

// per-thread pinned staging for the row copies (fill_block runs on many host threads)
struct Staging {
  void* buf = nullptr;
  size_t bytes = 0;
  cudaStream_t st = nullptr;
  int device = -1;
  ~Staging() {
    if (buf) cudaFreeHost(buf);
    if (st) cudaStreamDestroy(st);
  }
  cudaError_t get(int dev, size_t need) {
    cudaError_t e = cudaSuccess;
    if (device != dev) {
      if (st) cudaStreamDestroy(st);
      st = nullptr;
      device = dev;
    }
    if (!st && (e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking))) return e;
    if (bytes < need) {
      if (buf) cudaFreeHost(buf);
      buf = nullptr;
      bytes = 0;
      if ((e = cudaHostAlloc(&buf, need, cudaHostAllocDefault))) return e;
      bytes = need;
    }
    return e;
  }
};
thread_local Staging t_stage;

constexpr size_t kStageBytes = 64u << 20;

int get_plan(Collection& C, int lg, Plan** out) {
  auto it = C.plans.find(lg);
  if (it != C.plans.end()) {
    *out = &it->second;
    return PCF_OK;
  }
  Plan P;
  int64_t n = 0;
  const int rb = C.is_f32 ? 8 : 16;
  P.items.resize((size_t)std::max<int64_t>(1024, 4 * C.M));
  int rc = pcf_plan_pairwise(C.ss.data(), C.M, kPlanSmemBudget, 2048, lg, rb, P.items.data(),
                             (int64_t)P.items.size(), &n, &P.smem);
  if (rc == PCF_ERR_ARG && n > (int64_t)P.items.size()) {
    P.items.resize((size_t)n);
    rc = pcf_plan_pairwise(C.ss.data(), C.M, kPlanSmemBudget, 2048, lg, rb, P.items.data(), n, &n,
                           &P.smem);
  }
  if (rc) return rc;
  P.items.resize((size_t)n);
  cudaError_t e;
  if ((e = cudaMalloc((void**)&P.d_items, std::max<int64_t>(n, 1) * sizeof(pcf_work_item))) ||
      (e = cudaMemcpy(P.d_items, P.items.data(), n * sizeof(pcf_work_item),
                      cudaMemcpyHostToDevice)))
    return pfail(e, "pcf_collection plan upload");
  *out = &(C.plans[lg] = std::move(P));
  return PCF_OK;
}

// the whole matrix for `key` (caller holds C.mu)
int compute(Collection& C, const MatKey& key, std::shared_ptr<Matrix>* out) {
  Plan* P = nullptr;
  int rc = get_plan(C, key.lg, &P);
  if (rc) return rc;
  std::shared_ptr<Matrix> m;
  if (C.mat && C.mat.use_count() == 1) {
    m = C.mat;  // nobody is copying from the previous matrix: reuse its memory
  } else {
    m = std::make_shared<Matrix>();
    cudaError_t e = cudaMalloc((void**)&m->d, (size_t)C.M * (size_t)C.M * 8);
    if (e) return pfail(e, "pcf_collection matrix alloc");
  }
  C.mat.reset();
  m->key = key;
  cudaError_t e = launch_diag(C.d_recs, (const int64_t*)C.d_soff, (const int32_t*)C.d_perm, C.M,
                              key.op == PCF_OP_INNER, key.a, key.b, m->d, 0, C.M,
                              (unsigned long long*)C.d_err, C.st);
  if (e) return pfail(e, "pcf_collection diagonal");
  FillArgs A;
  A.recs = C.is_f32 ? C.d_tile : C.d_recs;
  A.recs8 = C.d_recsg;
  A.soff = (const int64_t*)C.d_soff;
  A.goff8 = (const int64_t*)C.d_goff;
  A.perm = (const int32_t*)C.d_perm;
  A.M = C.M;
  A.counter = (int*)C.d_cnt;
  A.op = key.op | (key.lg > 0 && key.op == PCF_OP_LP ? PCF_OP_FAST_POW : 0);
  A.p = key.p;
  A.a = key.a;
  A.b = key.b;
  A.apply_root = key.apply_root;
  A.out = m->d;
  A.out_f32 = 0;
  A.ld = C.M;
  A.err = (unsigned long long*)C.d_err;
  A.smem_bytes = P->smem;
  A.rec_bytes = C.is_f32 ? 8 : 16;
  int nsm = 0;
  A.num_sms = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, C.device) ==
                      cudaSuccess && nsm > 0 ? nsm : 148;
  const int64_t n = (int64_t)P->items.size();
  for (int64_t i = 0; i < n;) {
    int64_t j = i;
    while (j < n && P->items[j].smem_mode == P->items[i].smem_mode) ++j;
    A.items = P->d_items + i;
    A.n_items = (int)(j - i);
    A.smem_mode = P->items[i].smem_mode;
    if ((e = cudaMemsetAsync(C.d_cnt, 0, 4, C.st)) || (e = launch_fill_tiles(A, C.st)))
      return pfail(e, "pcf_collection fill");
    i = j;
  }
  if ((e = cudaStreamSynchronize(C.st))) return pfail(e, "pcf_collection fill sync");
  *out = C.mat = m;
  return PCF_OK;
}

template <typename T>
void write_block(const double* stage, int64_t w, int64_t c0, int64_t i0, int64_t i1,
                 const std::vector<int64_t>& jend, int diag, T* out, int64_t ld) {
  // rows: out[i, j0(i):jend(i)] (contiguous)
  for (int64_t i = i0; i < i1; ++i) {
    const int64_t j0 = diag ? i : i + 1;
    const double* src = stage + (i - i0) * w - c0;
    T* dst = out + i * ld;
    for (int64_t j = j0; j < jend[i - i0]; ++j) dst[j] = (T)src[j];
  }
  // mirrors: out[j, i] for the same (i, j), written row j by row j (contiguous in i),
  // 64-column tiles of the staged rows so the transposed reads stay in cache
  const int64_t jlo = diag ? i0 : i0 + 1;
  int64_t jhi = 0;
  for (int64_t i = i0; i < i1; ++i) jhi = std::max(jhi, jend[i - i0]);
  for (int64_t jb = jlo; jb < jhi; jb += 64) {
    const int64_t je = std::min(jb + 64, jhi);
    for (int64_t j = jb; j < je; ++j) {
      T* dst = out + j * ld;
      for (int64_t i = i0; i < i1; ++i) {
        const int64_t j0 = diag ? i : i + 1;
        if (j >= j0 && j < jend[i - i0]) dst[i] = (T)stage[(i - i0) * w + (j - c0)];
      }
    }
  }
}

}  // namespace
}  // namespace pcfb

using namespace pcfb;

extern "C" {

int pcf_collection_create(const void* tcat, const void* vcat, int is_f32, const int64_t* off,
                          int64_t M, void** handle) {
  if (!handle || !tcat || !vcat || !off || M < 1 || M > 0x7fffffff) {
    set_error("pcf_collection_create: bad arguments");
    return PCF_ERR_ARG;
  }
  *handle = nullptr;
  std::unique_ptr<Collection> C(new Collection());
  cudaError_t e = cudaGetDevice(&C->device);
  if (e) return pfail(e, "pcf_collection_create device");
  C->M = M;
  C->is_f32 = is_f32 ? 1 : 0;
  C->N = off[M] - off[0];
  std::vector<int64_t> sizes(M), off0(M + 1);
  for (int64_t i = 0; i < M; ++i) {
    sizes[i] = off[i + 1] - off[i];
    if (sizes[i] < 1) {
      set_error("pcf_collection_create: PCF %lld has no rows", (long long)i);
      return PCF_ERR_ARG;
    }
  }
  for (int64_t i = 0; i <= M; ++i) off0[i] = off[i] - off[0];
  C->perm.resize(M);
  std::iota(C->perm.begin(), C->perm.end(), 0);
  std::stable_sort(C->perm.begin(), C->perm.end(),
                   [&](int32_t x, int32_t y) { return sizes[x] > sizes[y]; });
  C->ss.resize(M);
  C->soff.assign(M + 1, 0);
  for (int64_t s = 0; s < M; ++s) {
    C->ss[s] = sizes[C->perm[s]];
    C->soff[s + 1] = C->soff[s] + C->ss[s];
  }
  const int GW = is_f32 ? 16 : 8;
  C->goff.resize((M + GW - 1) / GW + 1);
  int rc = pcf_group_offsets(C->ss.data(), M, GW, C->goff.data());
  if (rc) return rc;
  const size_t es = is_f32 ? 4 : 8;
  const int64_t N = C->N, ng = C->goff.back();
  void *d_t = nullptr, *d_v = nullptr, *d_off = nullptr;
  auto cleanup = [&]() {
    if (d_t) cudaFree(d_t);
    if (d_v) cudaFree(d_v);
    if (d_off) cudaFree(d_off);
  };
  if ((e = cudaStreamCreateWithFlags(&C->st, cudaStreamNonBlocking)) ||
      (e = cudaMalloc(&d_t, N * es)) || (e = cudaMalloc(&d_v, N * es)) ||
      (e = cudaMalloc(&d_off, (M + 1) * 8)) || (e = cudaMalloc(&C->d_perm, M * 4)) ||
      (e = cudaMalloc(&C->d_soff, (M + 1) * 8)) ||
      (e = cudaMalloc(&C->d_goff, C->goff.size() * 8)) ||
      (e = cudaMalloc(&C->d_recs, std::max<int64_t>(N, 1) * 16)) ||
      (e = cudaMalloc(&C->d_recsg, std::max<int64_t>(ng, 1) * (is_f32 ? 8 : 16))) ||
      (e = cudaMalloc(&C->d_err, 8)) || (e = cudaMalloc(&C->d_cnt, 64)) ||
      (is_f32 && (e = cudaMalloc(&C->d_tile, (N + 2) * 8)))) {
    cleanup();
    return pfail(e, "pcf_collection_create alloc");
  }
  if ((e = cudaMemcpyAsync(d_t, (const char*)tcat + off[0] * es, N * es, cudaMemcpyHostToDevice,
                           C->st)) ||
      (e = cudaMemcpyAsync(d_v, (const char*)vcat + off[0] * es, N * es, cudaMemcpyHostToDevice,
                           C->st)) ||
      (e = cudaMemcpyAsync(d_off, off0.data(), (M + 1) * 8, cudaMemcpyHostToDevice, C->st)) ||
      (e = cudaMemcpyAsync(C->d_perm, C->perm.data(), M * 4, cudaMemcpyHostToDevice, C->st)) ||
      (e = cudaMemcpyAsync(C->d_soff, C->soff.data(), (M + 1) * 8, cudaMemcpyHostToDevice,
                           C->st)) ||
      (e = cudaMemcpyAsync(C->d_goff, C->goff.data(), C->goff.size() * 8,
                           cudaMemcpyHostToDevice, C->st)) ||
      (e = cudaMemsetAsync(C->d_err, 0xff, 8, C->st))) {
    cudaStreamSynchronize(C->st);
    cleanup();
    return pfail(e, "pcf_collection_create upload");
  }
  if (!is_f32) {
    e = launch_pack(d_t, d_v, 0, (const int64_t*)d_off, (const int32_t*)C->d_perm,
                    (const int64_t*)C->d_soff, M, C->d_recs, (const int64_t*)C->d_goff,
                    C->d_recsg, C->st);
  } else {
    e = launch_pack(d_t, d_v, 1, (const int64_t*)d_off, (const int32_t*)C->d_perm,
                    (const int64_t*)C->d_soff, M, C->d_recs, nullptr, nullptr, C->st);
    if (!e) e = cudaMemsetAsync(C->d_tile, 0, (N + 2) * 8, C->st);
    if (!e)
      e = launch_pack32((const float*)d_t, (const float*)d_v, (const int64_t*)d_off,
                        (const int32_t*)C->d_perm, (const int64_t*)C->d_soff, M, C->d_tile,
                        (const int64_t*)C->d_goff, C->d_recsg, C->st);
  }
  cudaError_t e2 = cudaStreamSynchronize(C->st);
  cleanup();
  if (e || e2) return pfail(e ? e : e2, "pcf_collection_create pack");
  *handle = C.release();
  return PCF_OK;
}

void pcf_collection_free(void* handle) {
  if (!handle) return;
  Collection* C = (Collection*)handle;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(C->device);
  delete C;
  cudaSetDevice(prev);
}

int pcf_collection_fill_block(void* handle, int64_t r0, int64_t r1, int op, double p,
                              int apply_root, int diag, double a, double b, int32_t max_log2G,
                              void* out, int out_is_f32, int64_t ld, int64_t* err_i,
                              int64_t* err_j) {
  if (err_i) *err_i = -1;
  if (err_j) *err_j = -1;
  Collection* C = (Collection*)handle;
  if (!C || !out || r0 < 0 || r1 > (C ? C->M : 0) || ld < (C ? C->M : 0) ||
      (op != PCF_OP_LP && op != PCF_OP_INNER) || !(a >= 0.0) || !(a < b) || max_log2G < 0) {
    set_error("pcf_collection_fill_block: bad arguments");
    return PCF_ERR_ARG;
  }
  if (r1 <= r0) return PCF_OK;
  cudaError_t e = cudaSetDevice(C->device);
  if (e) return pfail(e, "pcf_collection_fill_block device");
  const int64_t M = C->M;
  MatKey key{op, apply_root ? 1 : 0, diag ? 1 : 0, max_log2G > 6 ? 6 : max_log2G,
             op == PCF_OP_INNER ? 0.0 : p, a, b};
  std::shared_ptr<Matrix> m;
  {
    std::lock_guard<std::mutex> lock(C->mu);
    if (!C->mat || !(C->mat->key == key)) {
      int rc = compute(*C, key, &m);
      if (rc) return rc;
    } else {
      m = C->mat;
    }
  }
  {  // transparent huge pages for the (usually fresh, np.zeros) result: the row and mirror
     // writes below are its first touch, and 2 MB pages fault 512x less often
    const size_t es = out_is_f32 ? 4 : 8;
    const uintptr_t b0 = ((uintptr_t)out + (2u << 20) - 1) & ~(uintptr_t)((2u << 20) - 1);
    const uintptr_t b1 = ((uintptr_t)out + (size_t)M * (size_t)ld * es) & ~(uintptr_t)((2u << 20) - 1);
    if (r0 == 0 && b1 > b0) madvise((void*)b0, b1 - b0, MADV_HUGEPAGE);
  }
  // rows [r0, r1), columns [c0, M): c0 = the block's first column that is written
  const int64_t c0 = diag ? r0 : std::min(r0 + 1, M);
  const int64_t w = M - c0;
  if (w <= 0) return PCF_OK;
  const int64_t rows_per = std::max<int64_t>(1, (int64_t)(kStageBytes / ((size_t)w * 8)));
  if ((e = t_stage.get(C->device, (size_t)std::min(rows_per, r1 - r0) * (size_t)w * 8)))
    return pfail(e, "pcf_collection_fill_block staging");
  std::vector<int64_t> jend;
  for (int64_t i0 = r0; i0 < r1; i0 += rows_per) {
    const int64_t i1 = std::min(i0 + rows_per, r1);
    if ((e = cudaMemcpy2DAsync(t_stage.buf, (size_t)w * 8, m->d + (size_t)i0 * M + c0,
                               (size_t)M * 8, (size_t)w * 8, (size_t)(i1 - i0),
                               cudaMemcpyDeviceToHost, t_stage.st)) ||
        (e = cudaStreamSynchronize(t_stage.st)))
      return pfail(e, "pcf_collection_fill_block copy");
    const double* stage = (const double*)t_stage.buf;
    // the block's first non-finite entry in row-major order ends it (pyx:109-112, 117-121)
    jend.assign((size_t)(i1 - i0), M);
    int64_t stop_i = -1, stop_j = -1;
    for (int64_t i = i0; i < i1 && stop_i < 0; ++i) {
      const double* row = stage + (i - i0) * w - c0;
      for (int64_t j = diag ? i : i + 1; j < M; ++j)
        if (!isfinite(row[j])) {
          stop_i = i;
          stop_j = j;
          break;
        }
    }
    const int64_t iw = stop_i >= 0 ? stop_i + 1 : i1;
    if (stop_i >= 0) jend[stop_i - i0] = stop_j;
    if (out_is_f32)
      write_block<float>(stage, w, c0, i0, iw, jend, diag, (float*)out, ld);
    else
      write_block<double>(stage, w, c0, i0, iw, jend, diag, (double*)out, ld);
    if (stop_i >= 0) {
      if (err_i) *err_i = stop_i;
      if (err_j) *err_j = stop_j;
      return PCF_OK;
    }
  }
  return PCF_OK;
}

}  // extern "C"
