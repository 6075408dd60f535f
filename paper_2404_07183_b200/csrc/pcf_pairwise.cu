// Pairwise rectangle-iteration engine: K1 (shared-memory tile kernel), K1r (one long row
// resident in shared memory), K1g (global-memory tiles for PCFs too long to stage), the fill_block row kernel, the pair list, the
// diagonal, and K3 (sort-pack).  See DESIGN.md for layouts and rooflines.
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
// The cells of the minimal common refinement of f and g on [a, b) are visited in time
// order, exactly as _accumulate does (pyx:37-59), except that a simultaneous jump
// (t_f == t_g) is taken as two steps, the second a zero-width cell [t, t) whose
// contribution h*0 = +-0 leaves the running sum bit-for-bit unchanged.  The step count is
// then a pure function of the sizes (N = (n_f-1-k0) + (n_g-1-m0)), so the loop needs no
// per-step termination test, and G lanes can split one pair along the merge path
// (diagonals d = lane*N/G, co-rank binary search).  G = 1 is the reference's strict
// left-to-right sum; G > 1 sums the same cell products in G contiguous runs that the
// caller adds in a fixed order.
//
// Each step issues ONE 16-byte load (the record of whichever cursor advances; the
// address and the destination registers are selected), so a warp's request covers all
// 32 lanes: shared-memory wavefronts are counted per quarter-warp, and a predicated
// two-load step would pay for eight quarter-phases instead of four.
//
// F and G are record pointers with strides SF / SG (records): the K1 row block is stored
// slot-interleaved (stride 8), columns and global data contiguously (stride 1).
// Bounded b: cell right edges are clamped to b (cells past b become zero-width) and the
// last lane adds the final cell h(v_f_last, v_g_last) * (b - t).  Unbounded b: the tail
// cell is left to the caller, which applies the divergence rule of pyx:47-51.
template <int HK, bool BOUNDED, int SF, int SG, typename RT = Rec>
__device__ __forceinline__ double lane_walk(const RT* __restrict__ F, int nf,
                                            const RT* __restrict__ Gv, int ng, int lane,
                                            int log2G, double p, double a, double b) {
  int k0 = 0, m0 = 0;
  if (a > 0.0) {  // start cursors k = max{i : t_i <= a} (pyx:33-36), by binary search
    k0 = upper_bound_count(nf - 1, a, [&](int x) { return F[x * SF].t; });
    m0 = upper_bound_count(ng - 1, a, [&](int x) { return Gv[x * SG].t; });
  }
  const RT* __restrict__ Fk = F + k0 * SF;
  const RT* __restrict__ Gm = Gv + m0 * SG;
  const int Nf = nf - 1 - k0, Ng = ng - 1 - m0;
  const int N = Nf + Ng;
  const int d0 = (int)(((long long)lane * N) >> log2G);
  const int d1 = (int)(((long long)(lane + 1) * N) >> log2G);
  // co-rank: number of f breakpoints among the first d0 merged breakpoints
  int lo = max(0, d0 - Ng), hi = min(d0, Nf);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (Fk[mid * SF].t <= Gm[(d0 - mid - 1) * SG].t) lo = mid + 1;
    else hi = mid;
  }
  const int i = lo, j = d0 - lo;
  double t;
  if (d0 == 0) {
    t = a;
  } else {
    const double tfp = i > 0 ? (double)Fk[(i - 1) * SF].t : 0.0;
    const double tgp = j > 0 ? (double)Gm[(j - 1) * SG].t : 0.0;
    t = fmax(tfp, tgp);
  }
  if (BOUNDED) t = fmin(t, b);
  // X/Y form: X is the cursor whose piece ends first, Y the other.  Every integrand here
  // is symmetric in (v_f, v_g), so the cell needs no f/g identity: tn = tX, advance X,
  // then swap roles if the new X piece outlasts Y.  (Ties may be taken in either order:
  // the extra zero-width cell adds +-0.)
  // The cursor state keeps the stored scalar kind (float for 8-byte records: half the
  // register moves per swap); every operand is widened to float64 before arithmetic.
  using ST = decltype(RT::t);
  const RT* __restrict__ xp = Fk + i * SF;
  const RT* __restrict__ yp = Gm + j * SG;
  int xs = SF, ys = SG;
  ST tx = xp->t, vx = xp->v, ty = yp->t, vy = yp->v;
  if (ty < tx) {
    const RT* tp = xp; xp = yp; yp = tp;
    int ts = xs; xs = ys; ys = ts;
    ST tt = tx; tx = ty; ty = tt;
    tt = vx; vx = vy; vy = tt;
  }
  // The current cell's integrand h(v_X, v_Y) is carried instead of v_X: after X advances
  // to (nt, nv) the next cell's integrand is h(nv, v_Y) whether or not the roles swap
  // (a swap makes the old Y the new X and nv the new Y; h is symmetric bit for bit), so
  // v_X never needs selecting.
  double acc = 0.0;
  double hc = hval<HK>((double)vx, (double)vy, p);
  const int steps = d1 - d0;
#pragma unroll 4
  for (int s = 0; s < steps; ++s) {
    double tn = (double)tx;
    if (BOUNDED) tn = fmin(tn, b);
    acc = __dadd_rn(acc, __dmul_rn(hc, __dsub_rn(tn, t)));
    t = tn;
    xp += xs;
    const ST nt = xp->t, nv = xp->v;
    hc = hval<HK>((double)nv, (double)vy, p);
    const bool sw = nt > ty;
    const RT* __restrict__ np = sw ? yp : xp;
    yp = sw ? xp : yp;
    xp = np;
    if (SF != SG) {
      const int ns = sw ? ys : xs;
      ys = sw ? xs : ys;
      xs = ns;
    }
    tx = sw ? ty : nt;
    ty = sw ? nt : ty;
    vy = sw ? nv : vy;
  }
  if (BOUNDED && (lane == (1 << log2G) - 1)) {
    acc = __dadd_rn(acc, __dmul_rn(hc, __dsub_rn(b, t)));
  }
  return acc;
}

// Finalise one entry: divergence rule, non-finite capture, root, cast, mirrored write
// (pyx:47-51, 109-116).  `hl` is h(v_f_last, v_g_last) (only used when unbounded).
template <bool BOUNDED, typename OutT>
__device__ __forceinline__ void finish_entry(double acc, double hl, double p, int apply_root,
                                             int64_t oi, int64_t oj, OutT* __restrict__ out,
                                             int64_t ld, int64_t M,
                                             unsigned long long* __restrict__ err) {
  double res = acc;
  if (!BOUNDED && hl != 0.0) res = hl > 0.0 ? INFINITY : -INFINITY;
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

// Completion signal of one work item (pcf_matrix_host's single-launch drain): called by
// thread 0 after a barrier that follows the item's last store; the copy stream waits for
// each chunk's counter (cuStreamWaitValue32) before copying its finished rows.
__device__ __forceinline__ void signal_item(const int32_t* __restrict__ tag,
                                            int32_t* __restrict__ done, int it) {
  __threadfence_system();
  atomicAdd(&done[tag[it]], 1);
}

// --------------------------------------------------------------------------------------
// K1: persistent tile kernel (512 threads, one CTA per SM).
//
// Work item = a block of 8*RG size-sorted rows x a column range.  The rows are staged
// once per item by one bulk copy from the slot-interleaved copy of the collection
// (recs8: record k of row u of an 8-row group at 16*(8k+u) -> shared-memory bank group
// u for every k); the columns stream through two shared-memory buffers of C contiguous
// PCFs (one bulk copy each, double-buffered on mbarriers).
//
// Lane mapping: a quarter-warp (8 lanes, the unit in which 16-byte shared loads are
// served) holds the 8 rows of one row group against ONE column: the row loads of a
// quarter always hit 8 distinct bank groups, so only column loads can conflict.
// 64 quarters = RG row groups x C columns x G merge-path segments.  With G > 1 the
// segment partials go through shared memory and one thread per pair adds them in
// segment order.
template <int HK, bool BOUNDED, typename OutT, typename RT, int GW>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_fill_tiles_smem(const RT* __restrict__ recs, const RT* __restrict__ recsg,
                      const int64_t* __restrict__ soff, const int64_t* __restrict__ goff,
                      const int32_t* __restrict__ perm, const PcfWorkItem* __restrict__ items,
                      int n_items, int* __restrict__ counter, double p, double a, double b,
                      int apply_root, OutT* __restrict__ out, int64_t ld, int64_t M,
                      unsigned long long* __restrict__ err,
                      const int32_t* __restrict__ item_tag, int32_t* __restrict__ tag_done) {
  // GW: rows per interleaved group = lanes per shared-memory phase for sizeof(RT)-byte
  // loads (8 x 16 B or 16 x 8 B = 128 B); CA: records per 16 B (bulk-copy granularity)
  constexpr int LOGGW = GW == 16 ? 4 : 3;
  constexpr int CA = 16 / (int)sizeof(RT);
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
  auto cstart = [&](int c0) { const int64_t r = soff[c0]; return r - r % CA; };
  auto cend = [&](int c1) { const int64_t r = soff[c1]; return (r + CA - 1) / CA * CA; };

  for (;;) {
    if (tid == 0) s_item = atomicAdd(counter, 1);
    __syncthreads();
    const int it = s_item;
    if (it >= n_items) break;
    const PcfWorkItem W = items[it];
    // logC bit 8: single-buffered columns (one chunk of twice the columns in flight, half
    // the merge-path segments; the planner picks it where G would otherwise be >= 16)
    const int logC = W.logC & 0xff;
    const bool single = (W.logC >> 8) & 1;
    const int logRG = W.nrows > GW ? 1 : 0;
    const int RG = 1 << logRG, C = 1 << logC, log2G = W.log2G, G = 1 << log2G;
    const int rg0 = W.row0 >> LOGGW;
    const int64_t rbase = goff[rg0];
    const uint32_t row_bytes = (uint32_t)((goff[rg0 + RG] - rbase) * sizeof(RT));
    const int nchunk = (W.col1 - W.col0 + C - 1) >> logC;
    const int c_first_end = min(W.col0 + C, W.col1);
    const uint32_t col_cap =
        (uint32_t)((cend(c_first_end) - cstart(W.col0)) * sizeof(RT)) + 16u;
    const uint32_t row_al = (row_bytes + 127u) & ~127u;
    const uint32_t col_al = (col_cap + 127u) & ~127u;
    unsigned char* rowbuf = smem;
    unsigned char* colbase = smem + row_al;  // column buffer k at colbase + k * col_al
    const int ncb = single ? 1 : 2;  // column buffers
    double* red = reinterpret_cast<double*>(smem + row_al + ncb * col_al);  // [2][512] partials
    double* redh = red + 2 * kTileThreads;                                   // [2][pairs] tails
    // issue chunk c into its column buffer (thread 0)
    auto issue = [&](int c) {
      const int cb = W.col0 + (c << logC), ce = min(cb + C, W.col1);
      const int64_t r0 = cstart(cb);
      const uint32_t nb = (uint32_t)((cend(ce) - r0) * sizeof(RT));
      const int kb = single ? 0 : (c & 1);
      fence_proxy_async();
      mbar_arrive_expect_tx(&bars[1 + kb], nb);
      bulk_g2s(colbase + kb * col_al, recs + r0, nb, &bars[1 + kb]);
    };

    if (tid == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&bars[0], row_bytes);
      bulk_g2s(rowbuf, recsg + rbase, row_bytes, &bars[0]);
      for (int c = 0; c < ncb && c < nchunk; ++c) issue(c);
    }
    // lane -> (row slot u, row group rho, column cc, segment g); fixed for the item
    const int u = tid & (GW - 1);
    const int Q = tid >> LOGGW;
    const int rho = Q & (RG - 1);
    const int cc = (Q >> logRG) & (C - 1);
    const int g = Q >> (logRG + logC);
    const int ps = W.row0 + GW * rho + u;
    const bool row_ok = ps < M;
    int nf = 0;
    const RT* F = reinterpret_cast<const RT*>(rowbuf) + (goff[rg0 + rho] - rbase) + u;
    int64_t oi = 0;
    if (row_ok) {
      nf = (int)(soff[ps + 1] - soff[ps]);
      oi = perm[ps];
    }
    const int pair_id = (cc * RG + rho) * GW + u;  // 0 .. GW*RG*C-1
    const int npairs = GW * RG * C;
    mbar_wait(&bars[0], ph_row);
    ph_row ^= 1u;

    for (int c = 0; c < nchunk; ++c) {
      const int buf = c & 1;                 // partials buffer (alternates every chunk)
      const int kb = single ? 0 : buf;       // column buffer
      const int cb = W.col0 + (c << logC);
      const int ce = min(cb + C, W.col1);
      const int qs = cb + cc;
      const bool ok = row_ok && qs < ce && qs > ps;
      mbar_wait(&bars[1 + kb], ph_col[kb]);
      ph_col[kb] ^= 1u;
      if (single && tid == 0 && c + 1 < nchunk) {
        // single buffer: the next chunk's copy can only start after this walk; warm L2
        const int nb0 = W.col0 + ((c + 1) << logC), ne = min(nb0 + C, W.col1);
        const int64_t r0 = cstart(nb0);
        bulk_prefetch_l2(recs + r0, (uint32_t)((cend(ne) - r0) * sizeof(RT)));
      }
      const RT* Gv = reinterpret_cast<const RT*>(colbase + kb * col_al);
      double acc = 0.0, hl = 0.0;
      if (ok) {
        const int ng = (int)(soff[qs + 1] - soff[qs]);
        Gv += soff[qs] - cstart(cb);
        acc = lane_walk<HK, BOUNDED, GW, 1, RT>(F, nf, Gv, ng, g, log2G, p, a, b);
        if (!BOUNDED) hl = hval<HK>(F[(nf - 1) * GW].v, Gv[ng - 1].v, p);
      }
      if (G == 1) {
        if (ok) finish_entry<BOUNDED, OutT>(acc, hl, p, apply_root, oi, perm[qs], out, ld, M, err);
        __syncthreads();  // column buffer `kb` is free again
        if (tid == 0 && c + ncb < nchunk) issue(c + ncb);
      } else {
        red[buf * kTileThreads + g * npairs + pair_id] = acc;  // segment-major: no conflicts
        if (g == 0) redh[buf * kTileThreads + pair_id] = hl;
        __syncthreads();  // partials visible, column buffer `kb` free again
        if (tid == 0 && c + ncb < nchunk) issue(c + ncb);  // before finishing: keep TMA busy
        if (tid < npairs) {
          const int pu = tid & (GW - 1), prho = (tid >> LOGGW) & (RG - 1);
          const int pcc = tid >> (LOGGW + logRG);
          const int pps = W.row0 + GW * prho + pu, pqs = cb + pcc;
          if (pps < M && pqs < ce && pqs > pps) {
            const double* r = red + buf * kTileThreads + tid;
            double s = r[0];
            for (int k = 1; k < G; ++k) s = __dadd_rn(s, r[k * npairs]);
            finish_entry<BOUNDED, OutT>(s, redh[buf * kTileThreads + tid], p, apply_root,
                                        perm[pps], perm[pqs], out, ld, M, err);
          }
        }
      }
    }
    __syncthreads();  // all finishers done before the next item reuses shared memory
    if (tag_done && tid == 0) signal_item(item_tag, tag_done, it);
  }
}

// K1c: one long row resident, interleaved column groups streamed -- K1 with the roles
// swapped, for rows too long for an 8-row group (c4's heavy tail).  A quarter-warp holds
// the GW columns of one interleaved group (recsg, the layout K1 stages its row groups in)
// against the row, so the column reads of a quarter hit GW distinct bank groups; only the
// row reads (lanes at unrelated positions of one PCF) can conflict.  64 quarters = CG
// groups per chunk x G merge-path segments; the groups stream through one or two shared
// buffers by bulk copy like K1's columns, the row is staged once per item.  Segment
// partials are added by one finishing thread per pair as in K1.
template <int HK, bool BOUNDED, typename OutT, typename RT, int GW>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_fill_colgroups(const RT* __restrict__ recs, const RT* __restrict__ recsg,
                     const int64_t* __restrict__ soff, const int64_t* __restrict__ goff,
                     const int32_t* __restrict__ perm, const PcfWorkItem* __restrict__ items,
                     int n_items, int* __restrict__ counter, double p, double a, double b,
                     int apply_root, OutT* __restrict__ out, int64_t ld, int64_t M,
                     unsigned long long* __restrict__ err,
                     const int32_t* __restrict__ item_tag, int32_t* __restrict__ tag_done) {
  constexpr int LOGGW = GW == 16 ? 4 : 3;
  constexpr int CA = 16 / (int)sizeof(RT);
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bars[3];  // 0: row, 1/2: column-group buffers
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
    const int logCG = W.logC & 0xff;
    const bool single = (W.logC >> 8) & 1;
    const int CG = 1 << logCG, log2G = W.log2G, G = 1 << log2G;
    const int ps = W.row0;
    const int nf = (int)(soff[ps + 1] - soff[ps]);
    const int64_t oi = perm[ps];
    const int64_t rlo = soff[ps] - soff[ps] % CA;
    const int64_t rhi = (soff[ps + 1] + CA - 1) / CA * CA;
    const uint32_t row_bytes = (uint32_t)((rhi - rlo) * sizeof(RT));
    const int gk0 = W.col0 >> LOGGW, gk1 = (W.col1 + GW - 1) >> LOGGW;
    const int nchunk = (gk1 - gk0 + CG - 1) >> logCG;
    const uint32_t col_cap =
        (uint32_t)((goff[min(gk0 + CG, gk1)] - goff[gk0]) * sizeof(RT));
    const uint32_t row_al = (row_bytes + 127u) & ~127u;
    const uint32_t col_al = (col_cap + 127u) & ~127u;
    const int ncb = single ? 1 : 2;
    unsigned char* rowbuf = smem;
    unsigned char* colbase = smem + row_al;
    double* red = reinterpret_cast<double*>(smem + row_al + ncb * col_al);  // [2][512] partials
    double* redh = red + 2 * kTileThreads;                                   // [2][pairs] tails
    auto issue = [&](int c) {
      const int kb0 = gk0 + (c << logCG), kb1 = min(kb0 + CG, gk1);
      const uint32_t nb = (uint32_t)((goff[kb1] - goff[kb0]) * sizeof(RT));
      const int kb = single ? 0 : (c & 1);
      fence_proxy_async();
      mbar_arrive_expect_tx(&bars[1 + kb], nb);
      bulk_g2s(colbase + kb * col_al, recsg + goff[kb0], nb, &bars[1 + kb]);
    };
    if (tid == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&bars[0], row_bytes);
      bulk_g2s(rowbuf, recs + rlo, row_bytes, &bars[0]);
      for (int c = 0; c < ncb && c < nchunk; ++c) issue(c);
    }
    const int u = tid & (GW - 1);
    const int Q = tid >> LOGGW;
    const int cg = Q & (CG - 1);
    const int g = Q >> logCG;
    const RT* F = reinterpret_cast<const RT*>(rowbuf) + (soff[ps] - rlo);
    const int pair_id = cg * GW + u;
    const int npairs = GW * CG;
    mbar_wait(&bars[0], ph_row);
    ph_row ^= 1u;
    for (int c = 0; c < nchunk; ++c) {
      const int buf = c & 1;
      const int kb = single ? 0 : buf;
      const int kbase = gk0 + (c << logCG);
      const int k = kbase + cg;
      const int64_t qs = (int64_t)k * GW + u;
      const bool ok = k < gk1 && qs >= W.col0 && qs < W.col1 && qs > ps && qs < M;
      mbar_wait(&bars[1 + kb], ph_col[kb]);
      ph_col[kb] ^= 1u;
      if (single && tid == 0 && c + 1 < nchunk) {  // warm L2 for the next chunk's copy
        const int nk0 = gk0 + ((c + 1) << logCG), nk1 = min(nk0 + CG, gk1);
        bulk_prefetch_l2(recsg + goff[nk0], (uint32_t)((goff[nk1] - goff[nk0]) * sizeof(RT)));
      }
      double acc = 0.0, hl = 0.0;
      if (ok) {
        const RT* Gv = reinterpret_cast<const RT*>(colbase + kb * col_al) +
                       (goff[k] - goff[kbase]) + u;
        const int ng = (int)(soff[qs + 1] - soff[qs]);
        acc = lane_walk<HK, BOUNDED, 1, GW, RT>(F, nf, Gv, ng, g, log2G, p, a, b);
        if (!BOUNDED) hl = hval<HK>(F[nf - 1].v, Gv[(ng - 1) * GW].v, p);
      }
      if (G == 1) {
        if (ok) finish_entry<BOUNDED, OutT>(acc, hl, p, apply_root, oi, perm[qs], out, ld, M, err);
        __syncthreads();
        if (tid == 0 && c + ncb < nchunk) issue(c + ncb);
      } else {
        red[buf * kTileThreads + g * npairs + pair_id] = acc;
        if (g == 0) redh[buf * kTileThreads + pair_id] = hl;
        __syncthreads();
        if (tid == 0 && c + ncb < nchunk) issue(c + ncb);
        if (tid < npairs) {
          const int pu = tid & (GW - 1), pcg = tid >> LOGGW;
          const int pk = kbase + pcg;
          const int64_t pqs = (int64_t)pk * GW + pu;
          if (pk < gk1 && pqs >= W.col0 && pqs < W.col1 && pqs > ps && pqs < M) {
            const double* r = red + buf * kTileThreads + tid;
            double sacc = r[0];
            for (int kk = 1; kk < G; ++kk) sacc = __dadd_rn(sacc, r[kk * npairs]);
            finish_entry<BOUNDED, OutT>(sacc, redh[buf * kTileThreads + tid], p, apply_root,
                                        oi, perm[pqs], out, ld, M, err);
          }
        }
      }
    }
    __syncthreads();
    if (tag_done && tid == 0) signal_item(item_tag, tag_done, it);
  }
}

// K1g: tiles whose PCFs are too long to stage; operands read straight from the
// contiguous records through L1/L2.  R x C pairs per pass, G lanes per pair in one warp
// (butterfly reduction).
template <int HK, bool BOUNDED, typename OutT, typename RT>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_fill_tiles_global(const RT* __restrict__ recs, const int64_t* __restrict__ soff,
                        const int32_t* __restrict__ perm, const PcfWorkItem* __restrict__ items,
                        int n_items, int* __restrict__ counter, double p, double a, double b,
                        int apply_root, OutT* __restrict__ out, int64_t ld, int64_t M,
                        unsigned long long* __restrict__ err,
                      const int32_t* __restrict__ item_tag, int32_t* __restrict__ tag_done) {
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
      const RT* F = recs + (row_ok ? soff[ps] : 0);
      const RT* Gv = recs + (ok ? soff[qs] : 0);
      int nf = 0, ng = 0;
      if (ok) {
        nf = (int)(soff[ps + 1] - soff[ps]);
        ng = (int)(soff[qs + 1] - soff[qs]);
        acc = lane_walk<HK, BOUNDED, 1, 1, RT>(F, nf, Gv, ng, lane, log2G, p, a, b);
      }
      for (int o = (1 << log2G) >> 1; o >= 1; o >>= 1)
        acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
      if (ok && lane == 0) {
        const double hl = BOUNDED ? 0.0 : hval<HK>(F[nf - 1].v, Gv[ng - 1].v, p);
        finish_entry<BOUNDED, OutT>(acc, hl, p, apply_root, (int64_t)perm[ps],
                                    (int64_t)perm[qs], out, ld, M, err);
      }
    }
    if (tag_done) {
      __syncthreads();
      if (tid == 0) signal_item(item_tag, tag_done, it);
    }
  }
}

// --------------------------------------------------------------------------------------
// K1r: row-resident tiles for rows too long for K1's 8-row groups (the heavy tail of c4).
//
// A work item is ONE size-sorted row x a column range.  The row is loaded into shared
// memory once per item and re-read by every pair of the item; the (shorter) columns are
// read through L1/L2.  For a long row against shorter columns almost every step of the
// walk advances the row cursor, so nearly all operand traffic lands in shared memory
// instead of costing one L1 line lookup per lane per step (K1g).  Lanes: C = 512/G
// columns x G merge-path segments, the G lanes of a pair contiguous in one warp.  Row
// loads from lanes at unrelated positions do conflict (random bank groups); the column
// share of the steps goes to L1.  G = 1 (exact mode) is the reference's left-to-right
// sum, bit for bit.
template <int HK, bool BOUNDED, typename OutT, typename RT>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_fill_rowres(const RT* __restrict__ recs, const int64_t* __restrict__ soff,
                  const int32_t* __restrict__ perm, const PcfWorkItem* __restrict__ items,
                  int n_items, int* __restrict__ counter, double p, double a, double b,
                  int apply_root, OutT* __restrict__ out, int64_t ld, int64_t M,
                  unsigned long long* __restrict__ err,
                      const int32_t* __restrict__ item_tag, int32_t* __restrict__ tag_done) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RT* rowS = reinterpret_cast<RT*>(smem_raw);
  __shared__ int s_item;
  const int tid = threadIdx.x;
  int cur_row = -1;
  for (;;) {
    if (tid == 0) s_item = atomicAdd(counter, 1);
    __syncthreads();  // also: every lane is done with the previous row
    const int it = s_item;
    if (it >= n_items) break;
    const PcfWorkItem W = items[it];
    const int ps = W.row0;
    const int nf = (int)(soff[ps + 1] - soff[ps]);
    if (ps != cur_row) {  // consecutive items of the same row keep it resident
      const RT* F = recs + soff[ps];
      for (int x = tid; x < nf; x += kTileThreads) rowS[x] = F[x];
      cur_row = ps;
    }
    __syncthreads();
    const int C = 1 << W.logC, log2G = W.log2G;
    const int cc = tid >> log2G;
    const int lane = tid & ((1 << log2G) - 1);
    for (int cb = max(W.col0, ps + 1); cb < W.col1; cb += C) {
      const int qs = cb + cc;
      const bool ok = qs < W.col1;
      double acc = 0.0;
      const RT* Gv = recs + (ok ? soff[qs] : 0);
      int ng = 0;
      if (ok) {
        ng = (int)(soff[qs + 1] - soff[qs]);
        acc = lane_walk<HK, BOUNDED, 1, 1, RT>(rowS, nf, Gv, ng, lane, log2G, p, a, b);
      }
      for (int o = (1 << log2G) >> 1; o >= 1; o >>= 1)
        acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
      if (ok && lane == 0) {
        const double hl = BOUNDED ? 0.0 : hval<HK>(rowS[nf - 1].v, Gv[ng - 1].v, p);
        finish_entry<BOUNDED, OutT>(acc, hl, p, apply_root, (int64_t)perm[ps],
                                    (int64_t)perm[qs], out, ld, M, err);
      }
    }
    if (tag_done) {
      __syncthreads();
      if (tid == 0) signal_item(item_tag, tag_done, it);
    }
  }
}

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
