// Pairwise engine, host-compiled part: the launch helpers for the tile kernels (device
// code in pcf_tiles.cuh: K1, K1c, K1r, K1g), the fill_block row kernel, the pair list, the
// diagonal, the sweep-cell enumerator and K3 (sort-pack).  See DESIGN.md for layouts and
// rooflines.
//
// Reference semantics being reproduced:
//   _sweepkern._accumulate  pkg/src/pcflib/_sweepkern.pyx:24-59  (per-pair walk)
//   _sweepkern.fill_block   pkg/src/pcflib/_sweepkern.pyx:88-121 (matrix fill, root, mirror)
//   _sweepkern.pack         pkg/src/pcflib/_sweepkern.pyx:72-85  (SoA concat + offsets)
#include "pcf_common.cuh"
#include "pcf_internal.h"
#include "pcf_tiles.cuh"
static_assert(pcfb::kRingSlots == pcfb::kK1sRingSlots, "K1s ring depth: planner and kernel disagree");
static_assert(pcfb::kRingThreads == pcfb::kK1sThreads, "K1s CTA size: planner and kernel disagree");

namespace pcfb {

// --------------------------------------------------------------------------------------
// Diagonal: Gram entries <f, f> (computed, pyx:104 with diag=True) or exact zeros for
// distances (never computed; matrix.py:163).  One thread per PCF, sequential walk;
// simultaneous jumps of f against itself take one step as in the reference.
template <bool BOUNDED>
__device__ __forceinline__ double self_inner(const Rec* __restrict__ F, int n, double a,
                                             double b) {
  int k = 0;
  if (a > 0.0) k = upper_bound_count(n - 1, a, [&](int x) { return F[x].t; });
  double t = a, acc = 0.0;
  for (;;) {
    const double tn = F[k].t, v = F[k].v;
    const double hv = __dmul_rn(v, v);
    if (tn >= b) {
      if (!BOUNDED) return (hv != 0.0) ? (hv > 0.0 ? INFINITY : -INFINITY) : acc;
      return __dadd_rn(acc, __dmul_rn(hv, __dsub_rn(b, t)));
    }
    acc = __dadd_rn(acc, __dmul_rn(hv, __dsub_rn(tn, t)));
    t = tn;
    ++k;
  }
}

template <bool BOUNDED, typename OutT>
__global__ void k_diag(const Rec* __restrict__ recs, const int64_t* __restrict__ soff,
                       const int32_t* __restrict__ perm, int64_t M, int gram, double a,
                       double b, OutT* __restrict__ out, int64_t ld,
                       unsigned long long* __restrict__ err) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < M;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = perm[s];
    if (!gram) {
      out[o * ld + o] = cast_out<OutT>(0.0);
      continue;
    }
    const double res =
        self_inner<BOUNDED>(recs + soff[s], (int)(soff[s + 1] - soff[s]), a, b);
    if (!isfinite(res)) atomicMin(err, (unsigned long long)(o * M + o));
    out[o * ld + o] = cast_out<OutT>(res);
  }
}

// --------------------------------------------------------------------------------------
// Row-range kernel mirroring fill_block(packed, r0, r1, ...) on ORIGINAL indices
// (pyx:88-121): rows [r0, r1), columns j > i (j >= i with diag).  One thread per entry,
// G = 1 (reference summation order), operands from global memory.  Output is a compact
// (r1-r0) x M row slab; the host mirrors it.
template <int HK, bool BOUNDED, typename OutT>
__global__ void k_fill_rows(const Rec* __restrict__ recs, const int64_t* __restrict__ soff,
                            const int32_t* __restrict__ inv, int64_t M, int64_t r0, int64_t r1,
                            int diag, double p, double a, double b, int apply_root,
                            OutT* __restrict__ slab, unsigned long long* __restrict__ err) {
  for (int64_t i = r0 + blockIdx.y; i < r1; i += gridDim.y) {
    const int64_t si = inv[i];
    const Rec* F = recs + soff[si];
    const int nf = (int)(soff[si + 1] - soff[si]);
    for (int64_t j = i + (diag ? 0 : 1) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M;
         j += (int64_t)gridDim.x * blockDim.x) {
      const int64_t sj = inv[j];
      const Rec* Gv = recs + soff[sj];
      const int ng = (int)(soff[sj + 1] - soff[sj]);
      double res;
      if (j == i) {
        if (HK == H_INNER) {
          res = self_inner<BOUNDED>(F, nf, a, b);
        } else {
          res = BOUNDED ? 0.0 : 0.0;  // |f - f|^p == 0 on every cell
        }
      } else {
        res = lane_walk<HK, BOUNDED, 1, 1>(F, nf, Gv, ng, 0, 0, p, a, b);
        if (!BOUNDED) {
          const double hl = hval<HK>(F[nf - 1].v, Gv[ng - 1].v, p);
          if (hl != 0.0) res = hl > 0.0 ? INFINITY : -INFINITY;
        }
      }
      if (!isfinite(res)) {
        atomicMin(err, (unsigned long long)(i * M + j));
      } else if (apply_root) {
        res = root_p(res, p);
      }
      slab[(i - r0) * M + j] = cast_out<OutT>(res);
    }
  }
}

// Raw (un-rooted) integral of explicit pairs (pair list), G = 1.  Used by the scalar
// integrate_pair entry point (pyx:62-69): returns +-inf on divergence like the reference.
template <int HK, bool BOUNDED>
__global__ void k_pair_list(const Rec* __restrict__ recs, const int64_t* __restrict__ soff,
                            const int64_t* __restrict__ pairs, int64_t npairs, double p, double a,
                            double b, double* __restrict__ res_out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < npairs;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t si = pairs[2 * k], sj = pairs[2 * k + 1];
    const Rec* F = recs + soff[si];
    const Rec* Gv = recs + soff[sj];
    const int nf = (int)(soff[si + 1] - soff[si]);
    const int ng = (int)(soff[sj + 1] - soff[sj]);
    double res = lane_walk<HK, BOUNDED, 1, 1>(F, nf, Gv, ng, 0, 0, p, a, b);
    if (!BOUNDED) {
      const double hl = hval<HK>(F[nf - 1].v, Gv[ng - 1].v, p);
      if (hl != 0.0) res = hl > 0.0 ? INFINITY : -INFINITY;
    }
    res_out[k] = res;
  }
}

// Cells of one sweep, in order (sweep.py:67-116): rectangles of the minimal common
// refinement of f and g on [a, b) (q >= 0; simultaneous jumps advance both cursors, no
// zero-width cells, the last right edge is b), or the segments of f alone (q < 0; pieces
// [t, t_next) while t_next < b, then [t, b)).  One thread; cells[4k..4k+3] =
// (l, r, v_f, v_g) (v_g = 0 for segments); *count = cells written.
__global__ void k_sweep_cells(const Rec* __restrict__ recs, const int64_t* __restrict__ soff,
                              int64_t s, int64_t q, double a, double b, double* __restrict__ cells,
                              int64_t cap, int64_t* __restrict__ count) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const Rec* F = recs + soff[s];
  const int nf = (int)(soff[s + 1] - soff[s]);
  int k = upper_bound_count(nf - 1, a, [&](int x) { return F[x].t; });
  double t = a;
  int64_t c = 0;
  auto emit = [&](double l, double r, double vf, double vg) {
    if (c < cap) {
      cells[4 * c] = l;
      cells[4 * c + 1] = r;
      cells[4 * c + 2] = vf;
      cells[4 * c + 3] = vg;
    }
    ++c;
  };
  if (q < 0) {
    while (k + 1 < nf && F[k].t < b) {
      emit(t, F[k].t, F[k].v, 0.0);
      t = F[k].t;
      ++k;
    }
    emit(t, b, F[k].v, 0.0);
  } else {
    const Rec* G = recs + soff[q];
    const int ng = (int)(soff[q + 1] - soff[q]);
    int m = upper_bound_count(ng - 1, a, [&](int x) { return G[x].t; });
    for (;;) {
      const double tnf = F[k].t, tng = G[m].t;
      const double tn = tnf < tng ? tnf : tng;
      if (tn >= b) {
        emit(t, b, F[k].v, G[m].v);
        break;
      }
      emit(t, tn, F[k].v, G[m].v);
      if (tnf == tn) ++k;
      if (tng == tn) ++m;
      t = tn;
    }
  }
  *count = c;
}

cudaError_t launch_sweep_cells(const void* recs, const int64_t* soff, int64_t s, int64_t q,
                               double a, double b, double* cells, int64_t cap, int64_t* count,
                               cudaStream_t st) {
  k_sweep_cells<<<1, 32, 0, st>>>((const Rec*)recs, soff, s, q, a, b, cells, cap, count);
  return cudaGetLastError();
}

// --------------------------------------------------------------------------------------
// K3: device-side pack.  Original-order SoA (tcat, vcat, off) -- the reference's pack()
// output, pyx:72-85 -- into size-sorted contiguous records and, optionally, the
// slot-interleaved 8-row-group copy (record k of sorted PCF s at goff8[s/8] + 8k + s%8).
// One warp per sorted PCF.
template <typename T>
__global__ void k_pack_sorted(const T* __restrict__ tcat, const T* __restrict__ vcat,
                              const int64_t* __restrict__ off, const int32_t* __restrict__ perm,
                              const int64_t* __restrict__ soff, int64_t M, Rec* __restrict__ recs,
                              const int64_t* __restrict__ goff8, Rec* __restrict__ recs8) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = w0; s < M; s += nw) {
    const int64_t o = perm[s];
    const int64_t src = off[o];
    const int64_t n = off[o + 1] - src;
    Rec* dst = recs + soff[s];
    Rec* dst8 = recs8 ? recs8 + goff8[s >> 3] + (s & 7) : nullptr;
    for (int64_t k = lane; k < n; k += 32) {
      Rec r;
      r.t = (k + 1 < n) ? (double)tcat[src + k + 1] : INFINITY;
      r.v = (double)vcat[src + k];
      dst[k] = r;
      if (dst8) dst8[8 * k] = r;
    }
  }
}

// float32 collections: 8-byte records, contiguous (+ CA-aligned tail) and slot-interleaved
// in groups of 16 (record k of sorted PCF s at goff16[s/16] + 16k + s%16).
__global__ void k_pack_sorted32(const float* __restrict__ tcat, const float* __restrict__ vcat,
                                const int64_t* __restrict__ off, const int32_t* __restrict__ perm,
                                const int64_t* __restrict__ soff, int64_t M,
                                Rec32* __restrict__ recs, const int64_t* __restrict__ goff16,
                                Rec32* __restrict__ recsg) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = w0; s < M; s += nw) {
    const int64_t o = perm[s];
    const int64_t src = off[o];
    const int64_t n = off[o + 1] - src;
    Rec32* dst = recs + soff[s];
    Rec32* dstg = recsg + goff16[s >> 4] + (s & 15);
    for (int64_t k = lane; k < n; k += 32) {
      Rec32 r;
      r.t = (k + 1 < n) ? tcat[src + k + 1] : INFINITY;
      r.v = vcat[src + k];
      dst[k] = r;
      dstg[16 * k] = r;
    }
  }
}

cudaError_t launch_pack32(const float* tcat, const float* vcat, const int64_t* off,
                          const int32_t* perm, const int64_t* soff, int64_t M, void* recs32,
                          const int64_t* goff16, void* recs32g, cudaStream_t st) {
  int grid = (int)((M * 32 + 255) / 256);
  if (grid > 148 * 64) grid = 148 * 64;
  if (grid < 1) grid = 1;
  k_pack_sorted32<<<grid, 256, 0, st>>>(tcat, vcat, off, perm, soff, M, (Rec32*)recs32, goff16,
                                        (Rec32*)recs32g);
  return cudaGetLastError();
}

// ======================================================================================
// launch helpers (called from the C-ABI layer)

template <int HK, bool BOUNDED, typename OutT>
static cudaError_t launch_tiles(const FillArgs& A, cudaStream_t st) {
  const int grid = A.num_sms;  // persistent: one CTA per SM
  if (A.smem_mode == 1) {
    cudaError_t e;
    if (A.rec_bytes == 8) {
      auto kern = k_fill_tiles_smem<HK, BOUNDED, OutT, Rec32, 16>;
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, A.smem_bytes);
      if (e != cudaSuccess) return e;
      kern<<<grid, kTileThreads, A.smem_bytes, st>>>(
          (const Rec32*)A.recs, (const Rec32*)A.recs8, A.soff, A.goff8, A.perm, A.items,
          A.n_items, A.counter, A.p, A.a, A.b, A.apply_root, (OutT*)A.out, A.ld, A.M, A.err, A.item_tag, A.tag_done);
    } else {
      auto kern = k_fill_tiles_smem<HK, BOUNDED, OutT, Rec, 8>;
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, A.smem_bytes);
      if (e != cudaSuccess) return e;
      kern<<<grid, kTileThreads, A.smem_bytes, st>>>(
          (const Rec*)A.recs, (const Rec*)A.recs8, A.soff, A.goff8, A.perm, A.items, A.n_items,
          A.counter, A.p, A.a, A.b, A.apply_root, (OutT*)A.out, A.ld, A.M, A.err, A.item_tag, A.tag_done);
    }
  } else if (A.smem_mode == 4) {  // K1s: exact mode, staged rows, columns through L1
    cudaError_t e;
    if (A.rec_bytes == 8) {
      auto kern = k_fill_rows_staged<HK, BOUNDED, OutT, Rec32, 16>;
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, A.smem_bytes);
      if (e != cudaSuccess) return e;
      kern<<<grid, kK1sThreads, A.smem_bytes, st>>>(
          (const Rec32*)A.recs, (const Rec32*)A.recs8, A.soff, A.goff8, A.perm, A.items,
          A.n_items, A.counter, A.p, A.a, A.b, A.apply_root, (OutT*)A.out, A.ld, A.M, A.err,
          A.item_tag, A.tag_done);
    } else {
      auto kern = k_fill_rows_staged<HK, BOUNDED, OutT, Rec, 8>;
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, A.smem_bytes);
      if (e != cudaSuccess) return e;
      kern<<<grid, kK1sThreads, A.smem_bytes, st>>>(
          (const Rec*)A.recs, (const Rec*)A.recs8, A.soff, A.goff8, A.perm, A.items, A.n_items,
          A.counter, A.p, A.a, A.b, A.apply_root, (OutT*)A.out, A.ld, A.M, A.err, A.item_tag,
          A.tag_done);
    }
  } else if (A.smem_mode == 3) {
    cudaError_t e;
    if (A.rec_bytes == 8) {
      auto kern = k_fill_colgroups<HK, BOUNDED, OutT, Rec32, 16>;
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, A.smem_bytes);
      if (e != cudaSuccess) return e;
      kern<<<grid, kTileThreads, A.smem_bytes, st>>>(
          (const Rec32*)A.recs, (const Rec32*)A.recs8, A.soff, A.goff8, A.perm, A.items,
          A.n_items, A.counter, A.p, A.a, A.b, A.apply_root, (OutT*)A.out, A.ld, A.M, A.err,
          A.item_tag, A.tag_done);
    } else {
      auto kern = k_fill_colgroups<HK, BOUNDED, OutT, Rec, 8>;
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, A.smem_bytes);
      if (e != cudaSuccess) return e;
      kern<<<grid, kTileThreads, A.smem_bytes, st>>>(
          (const Rec*)A.recs, (const Rec*)A.recs8, A.soff, A.goff8, A.perm, A.items, A.n_items,
          A.counter, A.p, A.a, A.b, A.apply_root, (OutT*)A.out, A.ld, A.M, A.err, A.item_tag,
          A.tag_done);
    }
  } else if (A.smem_mode == 2) {
    const size_t sm = (size_t)A.smem_bytes;
    cudaError_t e;
    if (A.rec_bytes == 8) {
      e = cudaFuncSetAttribute(k_fill_rowres<HK, BOUNDED, OutT, Rec32>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
      k_fill_rowres<HK, BOUNDED, OutT, Rec32><<<grid, kTileThreads, sm, st>>>(
          (const Rec32*)A.recs, A.soff, A.perm, A.items, A.n_items, A.counter, A.p, A.a, A.b,
          A.apply_root, (OutT*)A.out, A.ld, A.M, A.err, A.item_tag, A.tag_done);
    } else {
      e = cudaFuncSetAttribute(k_fill_rowres<HK, BOUNDED, OutT, Rec>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
      k_fill_rowres<HK, BOUNDED, OutT, Rec><<<grid, kTileThreads, sm, st>>>(
          (const Rec*)A.recs, A.soff, A.perm, A.items, A.n_items, A.counter, A.p, A.a, A.b,
          A.apply_root, (OutT*)A.out, A.ld, A.M, A.err, A.item_tag, A.tag_done);
    }
  } else if (A.rec_bytes == 8) {
    k_fill_tiles_global<HK, BOUNDED, OutT, Rec32><<<grid * 2, kTileThreads, 0, st>>>(
        (const Rec32*)A.recs, A.soff, A.perm, A.items, A.n_items, A.counter, A.p, A.a, A.b,
        A.apply_root, (OutT*)A.out, A.ld, A.M, A.err, A.item_tag, A.tag_done);
  } else {
    k_fill_tiles_global<HK, BOUNDED, OutT, Rec><<<grid * 2, kTileThreads, 0, st>>>(
        (const Rec*)A.recs, A.soff, A.perm, A.items, A.n_items, A.counter, A.p, A.a, A.b,
        A.apply_root, (OutT*)A.out, A.ld, A.M, A.err, A.item_tag, A.tag_done);
  }
  return cudaGetLastError();
}

template <bool BOUNDED, typename OutT>
static cudaError_t dispatch_hk(int hk, const FillArgs& A, cudaStream_t st) {
  switch (hk) {
    case H_L1: return launch_tiles<H_L1, BOUNDED, OutT>(A, st);
    case H_L2: return launch_tiles<H_L2, BOUNDED, OutT>(A, st);
    case H_L3: return launch_tiles<H_L3, BOUNDED, OutT>(A, st);
    case H_LP: return launch_tiles<H_LP, BOUNDED, OutT>(A, st);
    case H_LPX: return launch_tiles<H_LPX, BOUNDED, OutT>(A, st);
    default: return launch_tiles<H_INNER, BOUNDED, OutT>(A, st);
  }
}

int hkind_of(int op, double p) {
  if ((op & ~PCF_OP_FAST_POW) == PCF_OP_INNER) return H_INNER;
  if (p == 1.0) return H_L1;
  if (!(op & PCF_OP_FAST_POW)) return H_LPX;  // the reference's libm pow, bit for bit
  if (p == 2.0) return H_L2;
  if (p == 3.0) return H_L3;
  return H_LP;
}

cudaError_t launch_fill_tiles(const FillArgs& A, cudaStream_t st) {
  const int hk = hkind_of(A.op, A.p);
  const bool bounded = !isinf(A.b);
  if (A.out_f32) {
    return bounded ? dispatch_hk<true, float>(hk, A, st) : dispatch_hk<false, float>(hk, A, st);
  }
  return bounded ? dispatch_hk<true, double>(hk, A, st) : dispatch_hk<false, double>(hk, A, st);
}

cudaError_t launch_diag(const void* recs, const int64_t* soff, const int32_t* perm, int64_t M,
                        int gram, double a, double b, void* out, int out_f32, int64_t ld,
                        unsigned long long* err, cudaStream_t st) {
  const int threads = 256;
  int grid = (int)((M + threads - 1) / threads);
  if (grid > 65535) grid = 65535;
  if (grid < 1) grid = 1;
  const bool bounded = !isinf(b);
#define PCF_DIAG(BD, T)                                                                      \
  k_diag<BD, T><<<grid, threads, 0, st>>>((const Rec*)recs, soff, perm, M, gram, a, b, (T*)out, \
                                          ld, err)
  if (out_f32) {
    if (bounded) PCF_DIAG(true, float); else PCF_DIAG(false, float);
  } else {
    if (bounded) PCF_DIAG(true, double); else PCF_DIAG(false, double);
  }
#undef PCF_DIAG
  return cudaGetLastError();
}

template <int HK, bool BOUNDED, typename OutT>
static void launch_rows_t(const RowsArgs& A, cudaStream_t st) {
  dim3 block(128);
  int64_t cols = A.M;
  int gx = (int)((cols + 127) / 128);
  if (gx > 1024) gx = 1024;
  if (gx < 1) gx = 1;
  int64_t nrows = A.r1 - A.r0;
  int gy = (int)(nrows > 65535 ? 65535 : (nrows < 1 ? 1 : nrows));
  k_fill_rows<HK, BOUNDED, OutT><<<dim3(gx, gy), block, 0, st>>>(
      (const Rec*)A.recs, A.soff, A.inv, A.M, A.r0, A.r1, A.diag, A.p, A.a, A.b, A.apply_root,
      (OutT*)A.slab, A.err);
}

template <bool BOUNDED, typename OutT>
static void rows_hk(int hk, const RowsArgs& A, cudaStream_t st) {
  switch (hk) {
    case H_L1: launch_rows_t<H_L1, BOUNDED, OutT>(A, st); break;
    case H_L2: launch_rows_t<H_L2, BOUNDED, OutT>(A, st); break;
    case H_L3: launch_rows_t<H_L3, BOUNDED, OutT>(A, st); break;
    case H_LP: launch_rows_t<H_LP, BOUNDED, OutT>(A, st); break;
    case H_LPX: launch_rows_t<H_LPX, BOUNDED, OutT>(A, st); break;
    default: launch_rows_t<H_INNER, BOUNDED, OutT>(A, st); break;
  }
}

cudaError_t launch_fill_rows(const RowsArgs& A, cudaStream_t st) {
  const int hk = hkind_of(A.op, A.p);
  const bool bounded = !isinf(A.b);
  if (A.out_f32) {
    if (bounded) rows_hk<true, float>(hk, A, st); else rows_hk<false, float>(hk, A, st);
  } else {
    if (bounded) rows_hk<true, double>(hk, A, st); else rows_hk<false, double>(hk, A, st);
  }
  return cudaGetLastError();
}

cudaError_t launch_pair_list(const void* recs, const int64_t* soff, const int64_t* pairs,
                             int64_t npairs, int op, double p, double a, double b, double* res,
                             cudaStream_t st) {
  const int hk = hkind_of(op, p);
  const bool bounded = !isinf(b);
  int grid = (int)((npairs + 127) / 128);
  if (grid > 4096) grid = 4096;
  if (grid < 1) grid = 1;
#define PCF_PL(HK)                                                                              \
  do {                                                                                          \
    if (bounded)                                                                                \
      k_pair_list<HK, true><<<grid, 128, 0, st>>>((const Rec*)recs, soff, pairs, npairs, p, a, b, \
                                                  res);                                         \
    else                                                                                        \
      k_pair_list<HK, false><<<grid, 128, 0, st>>>((const Rec*)recs, soff, pairs, npairs, p, a,  \
                                                   b, res);                                     \
  } while (0)
  switch (hk) {
    case H_L1: PCF_PL(H_L1); break;
    case H_L2: PCF_PL(H_L2); break;
    case H_L3: PCF_PL(H_L3); break;
    case H_LP: PCF_PL(H_LP); break;
    case H_LPX: PCF_PL(H_LPX); break;
    default: PCF_PL(H_INNER); break;
  }
#undef PCF_PL
  return cudaGetLastError();
}

cudaError_t launch_pack(const void* tcat, const void* vcat, int f32, const int64_t* off,
                        const int32_t* perm, const int64_t* soff, int64_t M, void* recs,
                        const int64_t* goff8, void* recs8, cudaStream_t st) {
  int grid = (int)((M * 32 + 255) / 256);
  if (grid > 148 * 64) grid = 148 * 64;
  if (grid < 1) grid = 1;
  if (f32)
    k_pack_sorted<float><<<grid, 256, 0, st>>>((const float*)tcat, (const float*)vcat, off, perm,
                                               soff, M, (Rec*)recs, goff8, (Rec*)recs8);
  else
    k_pack_sorted<double><<<grid, 256, 0, st>>>((const double*)tcat, (const double*)vcat, off,
                                                perm, soff, M, (Rec*)recs, goff8, (Rec*)recs8);
  return cudaGetLastError();
}

}  // namespace pcfb
