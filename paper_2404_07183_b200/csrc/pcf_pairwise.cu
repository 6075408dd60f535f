// Pairwise rectangle-iteration engine (K1 tiles, K1g global-memory tiles, pair list,
// diagonal, sort-pack).  See DESIGN.md for the layout and the roofline.
//
// Reference semantics being reproduced:
//   _sweepkern._accumulate  pkg/src/pcflib/_sweepkern.pyx:24-59  (per-pair walk)
//   _sweepkern.fill_block   pkg/src/pcflib/_sweepkern.pyx:88-121 (matrix fill, root, mirror)
//   _sweepkern.pack         pkg/src/pcflib/_sweepkern.pyx:72-85  (SoA concat + offsets)
#include "pcf_common.cuh"
#include "pcf_internal.h"

namespace pcfb {

// --------------------------------------------------------------------------------------
// One lane's share of one pair's integral.
//
// The cells of the minimal common refinement of f and g on [a, b) are visited in
// time order, exactly as _accumulate does (pyx:37-59), except that a simultaneous
// jump (t_f == t_g) is taken as two steps: the f cursor first (stable merge order),
// then a zero-width cell [t, t) whose contribution h*0 = +-0 leaves the running sum
// bit-for-bit unchanged.  That makes the step count a pure function of the sizes
// (N = (n_f-1-k0) + (n_g-1-m0)) so the loop needs no per-step termination test, and
// lets G lanes split one pair along the merge path (diagonals d = lane*N/G) with a
// co-rank binary search.  G = 1 is the reference's strict left-to-right sum; G > 1
// sums the same cell products in G contiguous runs followed by a fixed butterfly.
//
// Bounded b: each cell's right edge is clamped to b (cells past b become zero-width),
// and the last lane adds the final cell h(v_f_last, v_g_last) * (b - t).
// Unbounded b: the tail cell is not accumulated; the caller applies the divergence
// rule of pyx:47-51 to the last values.
template <int HK, bool BOUNDED>
__device__ __forceinline__ double lane_walk(const Rec* __restrict__ F, int nf,
                                            const Rec* __restrict__ Gv, int ng, int lane,
                                            int log2G, double p, double a, double b) {
  int k0 = 0, m0 = 0;
  if (a > 0.0) {  // start cursors k = max{i : t_i <= a} (pyx:33-36), by binary search
    k0 = upper_bound_count(nf - 1, a, [&](int x) { return F[x].t; });
    m0 = upper_bound_count(ng - 1, a, [&](int x) { return Gv[x].t; });
  }
  const Rec* __restrict__ Fk = F + k0;
  const Rec* __restrict__ Gm = Gv + m0;
  const int Nf = nf - 1 - k0, Ng = ng - 1 - m0;
  const int N = Nf + Ng;
  const int d0 = (int)(((long long)lane * N) >> log2G);
  const int d1 = (int)(((long long)(lane + 1) * N) >> log2G);
  // co-rank: number of f breakpoints among the first d0 merged breakpoints.
  int lo = max(0, d0 - Ng), hi = min(d0, Nf);
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (Fk[mid].t <= Gm[d0 - mid - 1].t) lo = mid + 1;
    else hi = mid;
  }
  const int i = lo, j = d0 - lo;
  double t;
  if (d0 == 0) {
    t = a;
  } else {
    double tfp = i > 0 ? Fk[i - 1].t : 0.0;
    double tgp = j > 0 ? Gm[j - 1].t : 0.0;
    t = fmax(tfp, tgp);
  }
  if (BOUNDED) t = fmin(t, b);
  const Rec* __restrict__ fp = Fk + i;
  const Rec* __restrict__ gp = Gm + j;
  double tf = fp->t, vf = fp->v, tg = gp->t, vg = gp->v;
  double acc = 0.0;
  const int steps = d1 - d0;
#pragma unroll 4
  for (int s = 0; s < steps; ++s) {
    const bool af = tf <= tg;
    double tn = af ? tf : tg;
    if (BOUNDED) tn = fmin(tn, b);
    acc = __dadd_rn(acc, __dmul_rn(hval<HK>(vf, vg, p), __dsub_rn(tn, t)));
    t = tn;
    if (af) {
      ++fp;
      tf = fp->t;
      vf = fp->v;
    } else {
      ++gp;
      tg = gp->t;
      vg = gp->v;
    }
  }
  if (BOUNDED && (lane == (1 << log2G) - 1)) {
    acc = __dadd_rn(acc, __dmul_rn(hval<HK>(vf, vg, p), __dsub_rn(b, t)));
  }
  return acc;
}

// Finalise one entry: divergence rule, non-finite capture, root, cast, mirrored write.
// (pyx:47-51, 109-116).
template <int HK, bool BOUNDED, typename OutT>
__device__ __forceinline__ void finish_entry(double acc, double vf_last, double vg_last,
                                             double p, int apply_root, int64_t oi, int64_t oj,
                                             OutT* __restrict__ out, int64_t ld, int64_t M,
                                             unsigned long long* __restrict__ err) {
  double res = acc;
  if (!BOUNDED) {
    const double hl = hval<HK>(vf_last, vg_last, p);
    if (hl != 0.0) res = hl > 0.0 ? INFINITY : -INFINITY;
  }
  if (!isfinite(res)) {
    const int64_t lo = oi < oj ? oi : oj, hi = oi < oj ? oj : oi;
    atomicMin(err, (unsigned long long)(lo * M + hi));
  } else if (apply_root) {
    res = root_p(res, p);
  }
  const OutT o = cast_out<OutT>(res);
  out[oi * ld + oj] = o;
  out[oj * ld + oi] = o;
}

// --------------------------------------------------------------------------------------
// K1: persistent tile kernel.  Each work item is a row block (R size-sorted PCFs,
// staged once in shared memory by one bulk copy) against a column range streamed
// through a double-buffered shared-memory chunk of C PCFs (one bulk copy each).
// R*C pairs per chunk, G = 2^log2G lanes per pair (see lane_walk).
template <int HK, bool BOUNDED, typename OutT>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_fill_tiles_smem(const Rec* __restrict__ recs, const int64_t* __restrict__ soff,
                      const int32_t* __restrict__ perm, const PcfWorkItem* __restrict__ items,
                      int n_items, int* __restrict__ counter, double p, double a, double b,
                      int apply_root, OutT* __restrict__ out, int64_t ld, int64_t M,
                      unsigned long long* __restrict__ err) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bars[3];  // 0: rows, 1/2: column buffers
  __shared__ int s_item;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t ph_row = 0, ph_col[2] = {0u, 0u};

  for (;;) {
    if (tid == 0) s_item = atomicAdd(counter, 1);
    __syncthreads();
    const int it = s_item;
    if (it >= n_items) break;
    const PcfWorkItem W = items[it];
    const int R = W.nrows, C = 1 << W.logC, log2G = W.log2G;
    const int64_t rbase = soff[W.row0];
    const uint32_t row_bytes = (uint32_t)((soff[W.row0 + R] - rbase) * sizeof(Rec));
    const int nchunk = (W.col1 - W.col0 + C - 1) >> W.logC;
    const int c_first_end = min(W.col0 + C, W.col1);
    const uint32_t col_cap = (uint32_t)((soff[c_first_end] - soff[W.col0]) * sizeof(Rec));
    const uint32_t row_al = (row_bytes + 127u) & ~127u;
    const uint32_t col_al = (col_cap + 127u) & ~127u;
    unsigned char* rowbuf = smem;
    unsigned char* colbase = smem + row_al;  // column buffer k at colbase + k * col_al

    if (tid == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&bars[0], row_bytes);
      bulk_g2s(rowbuf, recs + rbase, row_bytes, &bars[0]);
      for (int c = 0; c < 2 && c < nchunk; ++c) {
        const int cb = W.col0 + (c << W.logC), ce = min(cb + C, W.col1);
        const uint32_t nb = (uint32_t)((soff[ce] - soff[cb]) * sizeof(Rec));
        mbar_arrive_expect_tx(&bars[1 + c], nb);
        bulk_g2s(colbase + c * col_al, recs + soff[cb], nb, &bars[1 + c]);
      }
    }
    // Per-thread pair coordinates are fixed for the whole item.
    const int pair = tid >> log2G;
    const int lane = tid & ((1 << log2G) - 1);
    const int r = pair >> W.logC;
    const int cc = pair & (C - 1);
    const bool row_ok = r < R;
    const int ps = W.row0 + r;
    int nf = 0;
    const Rec* F = reinterpret_cast<const Rec*>(rowbuf);
    int64_t oi = 0;
    if (row_ok) {
      nf = (int)(soff[ps + 1] - soff[ps]);
      F += soff[ps] - rbase;
      oi = perm[ps];
    }
    mbar_wait(&bars[0], ph_row);
    ph_row ^= 1u;

    for (int c = 0; c < nchunk; ++c) {
      const int buf = c & 1;
      const int cb = W.col0 + (c << W.logC);
      const int ce = min(cb + C, W.col1);
      const int qs = cb + cc;
      const bool ok = row_ok && qs < ce && qs > ps;
      mbar_wait(&bars[1 + buf], ph_col[buf]);
      ph_col[buf] ^= 1u;
      double acc = 0.0;
      int ng = 0;
      const Rec* Gv = reinterpret_cast<const Rec*>(colbase + buf * col_al);
      if (ok) {
        ng = (int)(soff[qs + 1] - soff[qs]);
        Gv += soff[qs] - soff[cb];
        acc = lane_walk<HK, BOUNDED>(F, nf, Gv, ng, lane, log2G, p, a, b);
      }
      for (int o = (1 << log2G) >> 1; o >= 1; o >>= 1)
        acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
      if (ok && lane == 0) {
        finish_entry<HK, BOUNDED, OutT>(acc, F[nf - 1].v, Gv[ng - 1].v, p, apply_root, oi,
                                        (int64_t)perm[qs], out, ld, M, err);
      }
      __syncthreads();  // buffer `buf` is free again
      if (tid == 0 && c + 2 < nchunk) {
        const int nb0 = W.col0 + ((c + 2) << W.logC), ne = min(nb0 + C, W.col1);
        const uint32_t nb = (uint32_t)((soff[ne] - soff[nb0]) * sizeof(Rec));
        fence_proxy_async();
        mbar_arrive_expect_tx(&bars[1 + buf], nb);
        bulk_g2s(colbase + buf * col_al, recs + soff[nb0], nb, &bars[1 + buf]);
      }
    }
  }
}

// K1g: same schedule, operands read straight from global memory (L1/L2).  Used for
// row blocks whose PCFs are too long for the shared-memory budget.
template <int HK, bool BOUNDED, typename OutT>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_fill_tiles_global(const Rec* __restrict__ recs, const int64_t* __restrict__ soff,
                        const int32_t* __restrict__ perm, const PcfWorkItem* __restrict__ items,
                        int n_items, int* __restrict__ counter, double p, double a, double b,
                        int apply_root, OutT* __restrict__ out, int64_t ld, int64_t M,
                        unsigned long long* __restrict__ err) {
  __shared__ int s_item;
  const int tid = threadIdx.x;
  for (;;) {
    if (tid == 0) s_item = atomicAdd(counter, 1);
    __syncthreads();
    const int it = s_item;
    __syncthreads();
    if (it >= n_items) break;
    const PcfWorkItem W = items[it];
    const int R = W.nrows, C = 1 << W.logC, log2G = W.log2G;
    const int pair = tid >> log2G;
    const int lane = tid & ((1 << log2G) - 1);
    const int r = pair >> W.logC;
    const int cc = pair & (C - 1);
    const bool row_ok = r < R;
    const int ps = W.row0 + r;
    for (int cb = W.col0; cb < W.col1; cb += C) {
      const int qs = cb + cc;
      const bool ok = row_ok && qs < W.col1 && qs > ps;
      double acc = 0.0;
      const Rec* F = recs + (row_ok ? soff[ps] : 0);
      const Rec* Gv = recs + (ok ? soff[qs] : 0);
      int nf = 0, ng = 0;
      if (ok) {
        nf = (int)(soff[ps + 1] - soff[ps]);
        ng = (int)(soff[qs + 1] - soff[qs]);
        acc = lane_walk<HK, BOUNDED>(F, nf, Gv, ng, lane, log2G, p, a, b);
      }
      for (int o = (1 << log2G) >> 1; o >= 1; o >>= 1)
        acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
      if (ok && lane == 0)
        finish_entry<HK, BOUNDED, OutT>(acc, F[nf - 1].v, Gv[ng - 1].v, p, apply_root,
                                        (int64_t)perm[ps], (int64_t)perm[qs], out, ld, M, err);
    }
  }
}

// --------------------------------------------------------------------------------------
// Diagonal: Gram entries <f, f> (computed, pyx:104 with diag=True) or exact zeros for
// distances (never computed; matrix.py:163).  One thread per PCF, sequential walk,
// simultaneous jumps of f against itself take one step as in the reference.
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
    const Rec* F = recs + soff[s];
    const int n = (int)(soff[s + 1] - soff[s]);
    int k = 0;
    if (a > 0.0) k = upper_bound_count(n - 1, a, [&](int x) { return F[x].t; });
    double t = a, acc = 0.0;
    double res;
    for (;;) {
      const double tn = F[k].t, v = F[k].v;
      const double hv = __dmul_rn(v, v);
      if (tn >= b) {
        if (!BOUNDED) {
          res = (hv != 0.0) ? (hv > 0.0 ? INFINITY : -INFINITY) : acc;
        } else {
          res = __dadd_rn(acc, __dmul_rn(hv, __dsub_rn(b, t)));
        }
        break;
      }
      acc = __dadd_rn(acc, __dmul_rn(hv, __dsub_rn(tn, t)));
      t = tn;
      ++k;
    }
    if (!isfinite(res)) atomicMin(err, (unsigned long long)(o * M + o));
    out[o * ld + o] = cast_out<OutT>(res);
  }
}

// --------------------------------------------------------------------------------------
// Row-range kernel mirroring fill_block(packed, r0, r1, ...) on ORIGINAL indices
// (pyx:88-121): rows [r0, r1), columns j > i (j >= i with diag).  One thread per
// entry, G = 1 (reference summation order), operands from global memory.  Output is a
// compact (r1-r0) x M row slab; the host mirrors it.
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
        // Gram diagonal: f against itself, one step per shared breakpoint.
        int k = 0;
        if (a > 0.0) k = upper_bound_count(nf - 1, a, [&](int x) { return F[x].t; });
        double t = a, acc = 0.0;
        for (;;) {
          const double tn = F[k].t, hv = hval<HK>(F[k].v, F[k].v, p);
          if (tn >= b) {
            if (!BOUNDED) res = (hv != 0.0) ? (hv > 0.0 ? INFINITY : -INFINITY) : acc;
            else res = __dadd_rn(acc, __dmul_rn(hv, __dsub_rn(b, t)));
            break;
          }
          acc = __dadd_rn(acc, __dmul_rn(hv, __dsub_rn(tn, t)));
          t = tn;
          ++k;
        }
      } else {
        res = lane_walk<HK, BOUNDED>(F, nf, Gv, ng, 0, 0, p, a, b);
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
    double res = lane_walk<HK, BOUNDED>(F, nf, Gv, ng, 0, 0, p, a, b);
    if (!BOUNDED) {
      const double hl = hval<HK>(F[nf - 1].v, Gv[ng - 1].v, p);
      if (hl != 0.0) res = hl > 0.0 ? INFINITY : -INFINITY;
    }
    res_out[k] = res;
  }
}

// --------------------------------------------------------------------------------------
// K3: device-side pack.  Original-order SoA (tcat, vcat, off) -- the reference's pack()
// output, pyx:72-85 -- into size-sorted records.  One warp per sorted PCF.
template <typename T>
__global__ void k_pack_sorted(const T* __restrict__ tcat, const T* __restrict__ vcat,
                              const int64_t* __restrict__ off, const int32_t* __restrict__ perm,
                              const int64_t* __restrict__ soff, int64_t M, Rec* __restrict__ recs) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = w0; s < M; s += nw) {
    const int64_t o = perm[s];
    const int64_t src = off[o];
    const int64_t n = off[o + 1] - src;
    Rec* dst = recs + soff[s];
    for (int64_t k = lane; k < n; k += 32) {
      Rec r;
      r.t = (k + 1 < n) ? (double)tcat[src + k + 1] : INFINITY;
      r.v = (double)vcat[src + k];
      dst[k] = r;
    }
  }
}

// ======================================================================================
// launch helpers (called from the C-ABI layer)

template <int HK, bool BOUNDED, typename OutT>
static cudaError_t launch_tiles(const FillArgs& A, cudaStream_t st) {
  const int nsm = A.num_sms;
  const int grid = nsm;  // persistent: one CTA per SM
  if (A.smem_mode) {
    auto kern = k_fill_tiles_smem<HK, BOUNDED, OutT>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, A.smem_bytes);
    if (e != cudaSuccess) return e;
    kern<<<grid, kTileThreads, A.smem_bytes, st>>>(
        (const Rec*)A.recs, A.soff, A.perm, A.items, A.n_items, A.counter, A.p, A.a, A.b,
        A.apply_root, (OutT*)A.out, A.ld, A.M, A.err);
  } else {
    k_fill_tiles_global<HK, BOUNDED, OutT><<<grid * 2, kTileThreads, 0, st>>>(
        (const Rec*)A.recs, A.soff, A.perm, A.items, A.n_items, A.counter, A.p, A.a, A.b,
        A.apply_root, (OutT*)A.out, A.ld, A.M, A.err);
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
    default: return launch_tiles<H_INNER, BOUNDED, OutT>(A, st);
  }
}

int hkind_of(int op, double p) {
  if (op == 1) return H_INNER;
  if (p == 1.0) return H_L1;
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
    default: PCF_PL(H_INNER); break;
  }
#undef PCF_PL
  return cudaGetLastError();
}

cudaError_t launch_pack(const void* tcat, const void* vcat, int f32, const int64_t* off,
                        const int32_t* perm, const int64_t* soff, int64_t M, void* recs,
                        cudaStream_t st) {
  int grid = (int)((M * 32 + 255) / 256);
  if (grid > 148 * 64) grid = 148 * 64;
  if (grid < 1) grid = 1;
  if (f32)
    k_pack_sorted<float><<<grid, 256, 0, st>>>((const float*)tcat, (const float*)vcat, off, perm,
                                               soff, M, (Rec*)recs);
  else
    k_pack_sorted<double><<<grid, 256, 0, st>>>((const double*)tcat, (const double*)vcat, off,
                                                perm, soff, M, (Rec*)recs);
  return cudaGetLastError();
}

}  // namespace pcfb
