// Pairwise tile kernels (device code): the lane walk, the entry finisher and the five
// persistent tile kernels K1 (k_fill_tiles_smem), K1c (k_fill_colgroups), K1g
// (k_fill_tiles_global), K1s (k_fill_rows_staged) and K1r (k_fill_rowres).  Included by pcf_pairwise.cu (nvcc, the
// op-coded integrands) and compiled again at run time by NVRTC with a user integrand
// (HK == H_USER, pcf_jit.cu) -- hence no host-only dependencies here.  See DESIGN.md.
//
// Reference semantics being reproduced:
//   _sweepkern._accumulate  pkg/src/pcflib/_sweepkern.pyx:24-59  (per-pair walk)
//   _sweepkern.fill_block   pkg/src/pcflib/_sweepkern.pyx:88-121 (matrix fill, root, mirror)
#pragma once
#include "pcf_common.cuh"

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
#ifndef PCF_K1_ICMP
#define PCF_K1_ICMP 0
#endif
#ifndef PCF_K1_UNROLL
#define PCF_K1_UNROLL 8
#endif
constexpr int kK1Unroll = PCF_K1_UNROLL;
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
#pragma unroll kK1Unroll
  for (int s = 0; s < steps; ++s) {
    double tn = (double)tx;
    if (BOUNDED) tn = fmin(tn, b);
    if constexpr (HK == H_USER) {
      // a user h may be non-finite on the (v_X', v_Y) pair of a tie's zero-width cell or
      // past b, which the reference never evaluates: skip those cells outright
      const double dt = __dsub_rn(tn, t);
      acc = __dadd_rn(acc, __dmul_rn(dt > 0.0 ? hc : 0.0, dt));
    } else {
      acc = __dadd_rn(acc, __dmul_rn(hc, __dsub_rn(tn, t)));
    }
    t = tn;
    xp += xs;
    const ST nt = xp->t, nv = xp->v;
    hc = hval<HK>((double)nv, (double)vy, p);
    bool sw;
    if constexpr (sizeof(ST) == 8 && PCF_K1_ICMP) {
      // record times are piece END times: > 0 or +inf, never NaN or -0, so the IEEE
      // order is the order of the bit patterns as signed integers (ALU, not the FP64 pipe)
      sw = __double_as_longlong((double)nt) > __double_as_longlong((double)ty);
    } else {
      sw = nt > ty;
    }
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
  if (BOUNDED && (lane == (1 << log2G) - 1) && (HK != H_USER || b > t)) {
    acc = __dadd_rn(acc, __dmul_rn(hc, __dsub_rn(b, t)));
  }
  return acc;
}

// Finalise one entry: divergence rule, non-finite capture, root, cast, mirrored write
// (pyx:47-51, 109-116).  `hl` is h(v_f_last, v_g_last) (only used when unbounded).
template <int HK, bool BOUNDED, typename OutT>
__device__ __forceinline__ void finish_entry(double acc, double hl, double p, int apply_root,
                                             int64_t oi, int64_t oj, OutT* __restrict__ out,
                                             int64_t ld, int64_t M,
                                             unsigned long long* __restrict__ err) {
  double res = acc;
  if (!BOUNDED && hl != 0.0) res = hl > 0.0 ? INFINITY : -INFINITY;
  if (!isfinite(res)) {
    const int64_t lo = oi < oj ? oi : oj, hi = oi < oj ? oj : oi;
    atomicMin(err, (unsigned long long)(lo * M + hi));
  } else if constexpr (HK == H_USER) {
    // CombinationIntegral.__call__ (integrate.py:197-203): round to the kind, then r
    if (apply_root) res = pcf_user_r((double)cast_out<OutT>(res));
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
    double* redh = red + 2 * kTileThreads;  // [2][npairs] tails (npairs = 512 / G)
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
    // Per-chunk global metadata (the lane's column size and offset in the chunk, the
    // output indices) is loaded one chunk ahead, so no warp starts a chunk's walk -- or a
    // finisher its stores -- behind an L2 round trip (long-scoreboard stalls at every chunk
    // start otherwise; all warps reach it together after the chunk barrier).
    const int fu = tid & (GW - 1), frho = (tid >> LOGGW) & (RG - 1);
    const int fcc = tid >> (LOGGW + logRG);
    const int fps = W.row0 + GW * frho + fu;   // finisher's row (G > 1, tid < npairs)
    const int64_t fpi = (G > 1 && tid < npairs && fps < M) ? (int64_t)perm[fps] : 0;
    int m_ng = 0, m_go = 0;
    int64_t m_pq = 0;
    auto load_meta = [&](int c) {
      const int cb = W.col0 + (c << logC), ce = min(cb + C, W.col1);
      const int qs = cb + cc;
      m_ng = 0; m_go = 0; m_pq = 0;
      if (row_ok && qs < ce && qs > ps && g < G) {
        const int64_t s0 = soff[qs];
        m_ng = (int)(soff[qs + 1] - s0);
        m_go = (int)(s0 - cstart(cb));
        if (G == 1) m_pq = perm[qs];
      }
      if (G > 1 && tid < npairs) {
        const int pqs = cb + fcc;
        if (fps < M && pqs < ce && pqs > fps) m_pq = perm[pqs];
      }
    };
    if (nchunk > 0) load_meta(0);
    mbar_wait(&bars[0], ph_row);
    ph_row ^= 1u;

    for (int c = 0; c < nchunk; ++c) {
      const int buf = c & 1;                 // partials buffer (alternates every chunk)
      const int kb = single ? 0 : buf;       // column buffer
      const int cb = W.col0 + (c << logC);
      const int ce = min(cb + C, W.col1);
      const int qs = cb + cc;
      // g >= G: an idle quarter (exact-mode items with fewer than 64 row x column lanes)
      const bool ok = row_ok && qs < ce && qs > ps && g < G;
      const int ng = m_ng, go = m_go;
      const int64_t pq = m_pq;
      if (c + 1 < nchunk) load_meta(c + 1);  // in flight during this chunk's walk
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
        Gv += go;
        acc = lane_walk<HK, BOUNDED, GW, 1, RT>(F, nf, Gv, ng, g, log2G, p, a, b);
        if (!BOUNDED && g == 0) hl = hval<HK>(F[(nf - 1) * GW].v, Gv[ng - 1].v, p);
      }
      if (G == 1) {
        if (ok) finish_entry<HK, BOUNDED, OutT>(acc, hl, p, apply_root, oi, pq, out, ld, M, err);
        __syncthreads();  // column buffer `kb` is free again
        if (tid == 0 && c + ncb < nchunk) issue(c + ncb);
      } else {
        red[buf * kTileThreads + g * npairs + pair_id] = acc;  // segment-major: no conflicts
        if (g == 0) redh[buf * npairs + pair_id] = hl;
        __syncthreads();  // partials visible, column buffer `kb` free again
        if (tid == 0 && c + ncb < nchunk) issue(c + ncb);  // before finishing: keep TMA busy
        if (tid < npairs) {
          const int pqs = cb + fcc;
          if (fps < M && pqs < ce && pqs > fps) {
            const double* r = red + buf * kTileThreads + tid;
            double s = r[0];
            for (int k = 1; k < G; ++k) s = __dadd_rn(s, r[k * npairs]);
            finish_entry<HK, BOUNDED, OutT>(s, redh[buf * npairs + tid], p, apply_root,
                                        fpi, pq, out, ld, M, err);
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
    double* redh = red + 2 * kTileThreads;  // [2][npairs] tails (npairs = 512 / G)
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
        if (!BOUNDED && g == 0) hl = hval<HK>(F[nf - 1].v, Gv[(ng - 1) * GW].v, p);
      }
      if (G == 1) {
        if (ok) finish_entry<HK, BOUNDED, OutT>(acc, hl, p, apply_root, oi, perm[qs], out, ld, M, err);
        __syncthreads();
        if (tid == 0 && c + ncb < nchunk) issue(c + ncb);
      } else {
        red[buf * kTileThreads + g * npairs + pair_id] = acc;
        if (g == 0) redh[buf * npairs + pair_id] = hl;
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
            finish_entry<HK, BOUNDED, OutT>(sacc, redh[buf * npairs + tid], p, apply_root,
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
        finish_entry<HK, BOUNDED, OutT>(acc, hl, p, apply_root, (int64_t)perm[ps],
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
// K1s: exact mode (G = 1) for row blocks whose 64 columns per chunk do not fit next to
// them.  The row block is staged as in K1 (interleaved groups, one bulk copy); the
// columns stay in global memory and reach each lane through a private prefetch ring in
// shared memory (kRingSlots records per lane, filled by per-thread cp.async = LDGSTS).
//
// Bank mapping: lane L holds row slot u = L % GW, whose records sit in bank group u of
// the interleaved row block.  Its ring slot k sits at
//   ring_base + (L / GW) * (kRingSlots * 128) + k * 128 + (L % GW) * sizeof(RT)
// -- bank group L % GW as well, for every k.  Every shared load of a lane (row record or
// ring slot) hits its own bank group, so a quarter-warp is ONE wavefront whatever
// positions its lanes are at (K1's shared column chunk pays ~2x in conflicts for that).
// The ring base is 1 KB aligned, so the next slot is one add and one LOP3 (bits 7-9 wrap).
//
// Latency: when a lane's column cursor advances it reads the next slot and refills the
// slot it leaves with the record kRingSlots ahead.  A record is therefore requested
// >= D - 1 walk steps before it is read; with one commit group per two steps,
// cp.async.wait_group((D - 3) / 2) before each pair of steps guarantees it landed while
// the last steps' requests stay in flight (~L2 latency hidden).
constexpr int kRingSlots = 8;
constexpr uint32_t kRingAlign = 1024;
// K1s CTA size: 20 warps (the other tile kernels use 512 threads); 8 rows x 80 columns per
// pass -- more warps to hide the shared-memory latency of the walk's dependent chain
constexpr int kRingThreads = 640;
#ifndef PCF_RING_L1
#define PCF_RING_L1 0
#endif
constexpr bool kRingL1 = PCF_RING_L1;
#ifndef PCF_RING_UNROLL
#define PCF_RING_UNROLL 2
#endif
constexpr int kRingUnroll = PCF_RING_UNROLL;  // step pairs per unrolled iteration  // refills through L1 (.ca): neighbours share a line

// The walk of one lane over merge-path segment `lane` of 2^log2G (G = 1: the whole pair,
// left to right -- the reference's sum) with the row in shared memory (stride SF records:
// GW for K1s's interleaved groups, 1 for K1r's contiguous row) and the column streamed
// through the lane's ring of D slots (slot k at ring + k * 128).
template <int HK, bool BOUNDED, typename RT, int D, int SF>
__device__ __forceinline__ double lane_walk_ring(const RT* __restrict__ F, int nf,
                                                 const RT* __restrict__ gcol, int ng,
                                                 uint32_t ring, int lane, int log2G, double p,
                                                 double a, double b) {
  using ST = decltype(RT::t);
  constexpr uint32_t RB = (uint32_t)sizeof(RT);
  constexpr uint32_t RS = SF * RB;           // row record stride (bytes)
  constexpr uint32_t CS = 128;               // ring slot stride
  constexpr uint32_t WRAP = (D - 1) * CS;    // slot-index bits of a ring address
  static_assert(D * CS <= kRingAlign && (D & (D - 1)) == 0, "ring slots");
  int k0 = 0, m0 = 0;
  if (a > 0.0) {  // start cursors k = max{i : t_i <= a} (pyx:33-36)
    k0 = upper_bound_count(nf - 1, a, [&](int x) { return (double)F[x * SF].t; });
    m0 = upper_bound_count(ng - 1, a, [&](int x) { return (double)gcol[x].t; });
  }
  const RT* __restrict__ Fk = F + k0 * SF;
  const RT* __restrict__ Gm = gcol + m0;
  const int Nf = nf - 1 - k0, Ng = ng - 1 - m0;
  const int N = Nf + Ng;
  const int d0 = (int)(((long long)lane * N) >> log2G);
  const int d1 = (int)(((long long)(lane + 1) * N) >> log2G);
  int i = 0;
  if (log2G > 0) {  // co-rank of diagonal d0 (see lane_walk); the column from L2
    int lo = max(0, d0 - Ng), hi = min(d0, Nf);
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (Fk[mid * SF].t <= Gm[d0 - mid - 1].t) lo = mid + 1;
      else hi = mid;
    }
    i = lo;
  }
  const int j = d0 - i;
  double t;
  if (d0 == 0) {
    t = a;
  } else {
    const double tfp = i > 0 ? (double)Fk[(i - 1) * SF].t : 0.0;
    const double tgp = j > 0 ? (double)Gm[j - 1].t : 0.0;
    t = fmax(tfp, tgp);
  }
  if (BOUNDED) t = fmin(t, b);
  const int steps = d1 - d0;
  const int jc0 = m0 + j;  // the lane's first column record
  const char* gb = reinterpret_cast<const char*>(gcol);
  const uint32_t boff_last = (uint32_t)(ng - 1) * RB;
  // the previous pair's in-flight prefetches must land before their slots are reused
  cp_async_wait<0>();
#pragma unroll
  for (int x = 0; x < D; ++x) {
    const uint32_t r = (uint32_t)min(jc0 + x, ng - 1);
    cp_async_rec<sizeof(RT)>(ring + (uint32_t)((jc0 + x) & (D - 1)) * CS, gb + r * RB);
  }
  cp_async_commit();
  cp_async_wait<0>();
  uint32_t boff = (uint32_t)min(jc0 + D, ng - 1) * RB;    // next record to request
  const uint32_t cslot = ring + (uint32_t)(jc0 & (D - 1)) * CS;  // the current column record
  // loop-carried: the slot of the NEXT column record.  The slot a column advance leaves
  // (refill target) is recomputed from it as a temporary, so no register an in-flight
  // LDGSTS still has to read is overwritten right after it (a WAR stall on the MIO queue)
  uint32_t cnext;
  asm("lop3.b32 %0, %1, %2, %3, 0xE2;" : "=r"(cnext) : "r"(cslot + CS), "n"(WRAP), "r"(cslot));
  uint32_t rnext = smem_u32(Fk + i * SF);
  ST tr, vr, tc, vc;
  lds_rec(rnext, tr, vr);
  lds_rec(cslot, tc, vc);
  rnext += RS;
  // X/Y walk (see lane_walk) with the column cursor's identity carried in xc: X is the
  // cursor whose piece ends first; when the roles swap, X becomes the other cursor.
  bool xc = tc < tr;
  ST tx = xc ? tc : tr, ty = xc ? tr : tc, vy = xc ? vr : vc;
  const ST vx = xc ? vc : vr;
  double acc = 0.0;
  double hc = hval<HK>((double)vx, (double)vy, p);
  auto step = [&]() {
    double tn = (double)tx;
    if (BOUNDED) tn = fmin(tn, b);
    if constexpr (HK == H_USER) {
      const double dt = __dsub_rn(tn, t);
      acc = __dadd_rn(acc, __dmul_rn(dt > 0.0 ? hc : 0.0, dt));
    } else {
      acc = __dadd_rn(acc, __dmul_rn(hc, __dsub_rn(tn, t)));
    }
    t = tn;
    const uint32_t addr = xc ? cnext : rnext;
    if (xc) {  // the column advances: refill the slot it leaves, D records ahead
      uint32_t left, nn;  // ((x +- CS) & WRAP) | (x & ~WRAP): one LOP3 each
      asm("lop3.b32 %0, %1, %2, %3, 0xE2;" : "=r"(left) : "r"(cnext + (D - 1) * CS), "n"(WRAP), "r"(cnext));
      asm("lop3.b32 %0, %1, %2, %3, 0xE2;" : "=r"(nn) : "r"(cnext + CS), "n"(WRAP), "r"(cnext));
      cp_async_rec<sizeof(RT), kRingL1>(left, gb + boff);
      boff = min(boff + RB, boff_last);
      cnext = nn;
    } else {
      rnext += RS;
    }
    ST nt, nv;
    lds_rec(addr, nt, nv);
    hc = hval<HK>((double)nv, (double)vy, p);
    const bool sw = nt > ty;
    tx = sw ? ty : nt;
    ty = sw ? nt : ty;
    vy = sw ? nv : vy;
    xc = xc != sw;
  };
  int s = 0;
  if constexpr (D >= 8) {
    // one commit group per two steps: a record read at step s was requested at step
    // <= s - (D - 1), i.e. in a group at least 3 groups old, so waiting until <= 2 groups
    // are pending before each pair of steps covers both
#pragma unroll kRingUnroll
    for (; s + 1 < steps; s += 2) {
      cp_async_wait<(D - 3) / 2>();
      step();
      step();
      cp_async_commit();
    }
  }
#pragma unroll 2
  for (; s < steps; ++s) {  // one group per step: requested >= D - 1 steps before
    cp_async_wait<(D >= 8 ? (D - 3) / 2 : D - 2)>();  // (after pairs: groups of two steps)
    step();
    cp_async_commit();
  }
  if (BOUNDED && (lane == (1 << log2G) - 1) && (HK != H_USER || b > t))
    acc = __dadd_rn(acc, __dmul_rn(hc, __dsub_rn(b, t)));
  return acc;
}

template <int HK, bool BOUNDED, typename OutT, typename RT, int GW>
__global__ void __launch_bounds__(kRingThreads, 1)
    k_fill_rows_staged(const RT* __restrict__ recs, const RT* __restrict__ recsg,
                       const int64_t* __restrict__ soff, const int64_t* __restrict__ goff,
                       const int32_t* __restrict__ perm, const PcfWorkItem* __restrict__ items,
                       int n_items, int* __restrict__ counter, double p, double a, double b,
                       int apply_root, OutT* __restrict__ out, int64_t ld, int64_t M,
                       unsigned long long* __restrict__ err,
                       const int32_t* __restrict__ item_tag, int32_t* __restrict__ tag_done) {
  constexpr int LOGGW = GW == 16 ? 4 : 3;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ int s_item;
  const int tid = threadIdx.x;
  // the prefetch rings at the top of the dynamic shared memory (1 KB aligned); this
  // lane's slot 0
  const uint32_t ring =
      ((smem_u32(smem) + dynamic_smem_bytes() -
        (uint32_t)(kRingSlots * kRingThreads * sizeof(RT))) & ~(kRingAlign - 1)) +
      (uint32_t)(tid / GW) * (kRingSlots * 128u) + (uint32_t)(tid % GW) * (uint32_t)sizeof(RT);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t ph = 0;
  for (;;) {
    if (tid == 0) s_item = atomicAdd(counter, 1);
    __syncthreads();
    const int it = s_item;
    if (it >= n_items) break;
    const PcfWorkItem W = items[it];
    const int logRG = W.nrows > GW ? 1 : 0;
    const int RG = 1 << logRG, C = (kRingThreads / GW) >> logRG;  // columns per pass
    const int rg0 = W.row0 >> LOGGW;
    const int64_t rbase = goff[rg0];
    const uint32_t row_bytes = (uint32_t)((goff[rg0 + RG] - rbase) * sizeof(RT));
    if (tid == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&bar, row_bytes);
      bulk_g2s(smem, recsg + rbase, row_bytes, &bar);
    }
    const int u = tid & (GW - 1);
    const int Q = tid >> LOGGW;
    const int rho = Q & (RG - 1);
    const int cc = Q >> logRG;
    const int ps = W.row0 + GW * rho + u;
    const bool row_ok = ps < M;
    const RT* F = reinterpret_cast<const RT*>(smem) + (goff[rg0 + rho] - rbase) + u;
    int nf = 0;
    int64_t oi = 0;
    if (row_ok) {
      nf = (int)(soff[ps + 1] - soff[ps]);
      oi = perm[ps];
    }
    mbar_wait(&bar, ph);
    ph ^= 1u;
    for (int cb = W.col0; cb < W.col1; cb += C) {
      const int qs = cb + cc;
      if (row_ok && qs < W.col1 && qs > ps) {
        const RT* Gv = recs + soff[qs];
        const int ng = (int)(soff[qs + 1] - soff[qs]);
        const double acc =
            lane_walk_ring<HK, BOUNDED, RT, kRingSlots, GW>(F, nf, Gv, ng, ring, 0, 0, p, a, b);
        const double hl = BOUNDED ? 0.0 : hval<HK>((double)F[(nf - 1) * GW].v,
                                                   (double)Gv[ng - 1].v, p);
        finish_entry<HK, BOUNDED, OutT>(acc, hl, p, apply_root, oi, perm[qs], out, ld, M, err);
      }
    }
    cp_async_wait<0>();  // no prefetch may land in the ring after the kernel moves on
    __syncthreads();  // every lane done with the rows before the next item's copy
    if (tag_done && tid == 0) signal_item(item_tag, tag_done, it);
  }
}

// --------------------------------------------------------------------------------------
// K1r: row-resident tiles for rows too long for K1's 8-row groups (the heavy tail of c4).
//
// A work item is ONE size-sorted row x a column range.  The row is loaded into shared
// memory once per item and re-read by every pair of the item; the (long) columns stream
// through each lane's prefetch ring (lane_walk_ring, as in K1s: cp.async refills kRingSlots
// records ahead; 4 slots for the few rows too long to leave room for 8 -- item flag
// logC bit 9).  Lanes: C = 512/G columns x G merge-path segments, the G lanes of a pair
// contiguous in one warp.  Row loads from lanes at unrelated positions do conflict (random
// bank groups); ring loads do not.  G = 1 (exact mode) is the reference's left-to-right
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
  constexpr int GWL = 128 / (int)sizeof(RT);  // lanes per 128-byte ring slot row
  const int tid = threadIdx.x;
  const uint32_t top = smem_u32(smem_raw) + dynamic_smem_bytes();
  int cur_row = -1;
  for (;;) {
    cp_async_wait<0>();  // no ring refill may still be landing when the row is replaced
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
    const bool small_ring = (W.logC >> 9) & 1;
    const int D = small_ring ? 4 : kRingSlots;
    const uint32_t ring = ((top - (uint32_t)(D * kTileThreads * sizeof(RT))) & ~(kRingAlign - 1)) +
                          (uint32_t)(tid / GWL) * (uint32_t)(D * 128) +
                          (uint32_t)(tid % GWL) * (uint32_t)sizeof(RT);
    const int C = 1 << (W.logC & 0xff), log2G = W.log2G;
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
        acc = small_ring
                  ? lane_walk_ring<HK, BOUNDED, RT, 4, 1>(rowS, nf, Gv, ng, ring, lane, log2G,
                                                          p, a, b)
                  : lane_walk_ring<HK, BOUNDED, RT, kRingSlots, 1>(rowS, nf, Gv, ng, ring, lane,
                                                                   log2G, p, a, b);
      }
      for (int o = (1 << log2G) >> 1; o >= 1; o >>= 1)
        acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
      if (ok && lane == 0) {
        const double hl = BOUNDED ? 0.0 : hval<HK>(rowS[nf - 1].v, Gv[ng - 1].v, p);
        finish_entry<HK, BOUNDED, OutT>(acc, hl, p, apply_root, (int64_t)perm[ps],
                                    (int64_t)perm[qs], out, ld, M, err);
      }
    }
    if (tag_done) {
      __syncthreads();
      if (tid == 0) signal_item(item_tag, tag_done, it);
    }
  }
}


}  // namespace pcfb
