// Tiled reduction-tree level (K5 / K7, v3): one CTA per tile of LT candidate positions.
//
// A level maps input nodes to output nodes (output k merges input nodes src[k], src[k]+1,
// or passes src[k] through when cnt[k] == 1 -- reduce.py:189-208).  Output node k's
// merge candidates occupy exactly the input positions of its input nodes, so a tile of
// candidate positions [e0, e0+LT) touches one or a few nodes ("segments").  Per tile:
//
//   1. build the segment table (node, candidate sub-range, co-ranks at the sub-range
//      ends -- binary searches only for the two partial segments at the tile edges);
//   2. stage every segment's A and B input windows (+1 element either side for the
//      previous-cell value and the tie checks) in shared memory with coalesced loads;
//   3. each thread walks LPT consecutive positions from shared memory ONCE, producing
//      the combined value and reduce_pair's keep flag (value changed w.r.t. the previous
//      cell; duplicate breakpoints dropped; passthrough nodes kept verbatim) into
//      registers;
//   4. block scan of the keep counts, decoupled look-back for the tile's output offset;
//   5. each thread stores its kept points.
//
// Single pass: every input point is read once and every output point written once
// (HBM traffic per level = 2 x 16 B per point for float64, the algorithmic minimum).
// Tiles whose nodes need several rounds (more than MAXSEG nodes) park their kept points
// in a scratch region until the offset is known.  Node start offsets are stored
// tile-relative and fixed up by k_fix_offsets.
#include <type_traits>
#include "pcf_common.cuh"
#include "pcf_internal.h"

namespace pcfb {
namespace lvl {

constexpr int LTH = 256;         // threads per tile CTA
constexpr int LPT = 8;           // positions per thread
constexpr int LT = LTH * LPT;    // candidate positions per tile
constexpr int MAXSEG = 64;       // node segments per round
// staged elements per round (both windows, +1 element either side, plus the 16-byte
// granule padding of the bulk copies: U - 1 elements at each end of each window)
template <typename T>
__host__ __device__ constexpr int wcap() { return LT + (4 + 4 * (16 / (int)sizeof(T) - 1)) * MAXSEG; }

enum { K_ADD = 0, K_MAX = 1, K_MIN = 2, K_MUL = 3, K_MOM = 4 };

template <int K>
__device__ __forceinline__ double vop(double x, double y) {
  if (K == K_ADD) return __dadd_rn(x, y);
  if (K == K_MUL) return __dmul_rn(x, y);
  if (K == K_MAX) return x > y ? x : y;  // Python max(x, y)
  return y < x ? y : x;                    // Python min(x, y)
}

template <typename T> __device__ __forceinline__ T to_t(double x);
template <> __device__ __forceinline__ double to_t<double>(double x) { return x; }
template <> __device__ __forceinline__ float to_t<float>(double x) { return __double2float_rn(x); }

struct Seg {
  int64_t node;   // output node
  int64_t base;   // input position of the node's A[0] (= first candidate position)
  int64_t na, nb;
  int64_t m0, m1;          // candidate sub-range within the node
  int64_t i0, j0, i1, j1;  // co-ranks at m0 and m1
  int64_t ia_lo, jb_lo;    // first staged A / B index
  int64_t ga, gb;          // global positions of the first staged A / B element
  int aoff, boff;          // shared-memory offsets of the staged windows
  int alen, blen;
  int pass;                // passthrough node
  double wB, wAB;          // moments weights nB/n, nA*nB/n
};

template <typename T>
__device__ __forceinline__ int64_t corank_g(const T* __restrict__ ta, int64_t na,
                                            const T* __restrict__ tb, int64_t nb, int64_t m) {
  int64_t lo = m > nb ? m - nb : 0, hi = m < na ? m : na;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ta[mid] <= tb[m - mid - 1]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <typename T, int K>
__global__ void __launch_bounds__(LTH, K == K_MOM ? 3 : 4)
    k_level_tiled(const T* __restrict__ t, const void* __restrict__ v_,
                  const double* __restrict__ v2, const int64_t* __restrict__ off,
                  const int64_t* __restrict__ src, const int32_t* __restrict__ cnt,
                  const int64_t* __restrict__ leaves, int64_t nout, int64_t ntot,
                  const int64_t* __restrict__ tile_node, const int64_t* __restrict__ tile_i,
                  int* __restrict__ tile_counter, unsigned long long* __restrict__ tile_status,
                  T* __restrict__ t_out, void* __restrict__ v_out_, double* __restrict__ v2_out,
                  int64_t* __restrict__ off_out, int32_t* __restrict__ status,
                  int64_t* __restrict__ tile_excl, T* __restrict__ x_t, void* __restrict__ x_v_,
                  double* __restrict__ x_v2) {
  using VT = typename std::conditional<K == K_MOM, double, T>::type;
  const VT* __restrict__ v = reinterpret_cast<const VT*>(v_);
  VT* __restrict__ v_out = reinterpret_cast<VT*>(v_out_);
  VT* __restrict__ x_v = reinterpret_cast<VT*>(x_v_);
  constexpr bool MOM = (K == K_MOM);

  __shared__ Seg seg[MAXSEG];
  __shared__ int seg_pos[MAXSEG + 1];  // round-relative candidate start of each segment
  extern __shared__ __align__(16) unsigned char dyn[];
  constexpr int WCAP = wcap<T>();
  constexpr int U = 16 / (int)sizeof(T);  // elements per 16-byte bulk-copy granule
  VT* s_v = reinterpret_cast<VT*>(dyn);                          // [WCAP]
  double* s_v2 = reinterpret_cast<double*>(dyn + WCAP * sizeof(VT));  // [WCAP] (moments)
  T* s_t = reinterpret_cast<T*>(dyn + WCAP * sizeof(VT) + (MOM ? WCAP * sizeof(double) : 0));
  __shared__ uint64_t s_bar;  // bulk-copy completion of the staged windows
  __shared__ int64_t s_next_node, s_round_end, s_tile, s_excl;
  __shared__ int scan_ws[LTH / 32];

  const int tid = threadIdx.x;
  // Tiles are taken in order from an atomic counter, so every tile's predecessors are
  // running or done -- the decoupled look-back below cannot wait on an unscheduled CTA.
  if (tid == 0) {
    s_tile = atomicAdd(tile_counter, 1);
    mbar_init(&s_bar, 1);
    fence_mbar_init();
  }
  uint32_t bar_phase = 0;
  __syncthreads();
  const int64_t tile = s_tile;
  // `ntot` is a host-side upper bound (the previous level's size); the live point count
  // is the end of the last output node's input range.  Tiles past it are empty.
  ntot = off[src[nout - 1] + cnt[nout - 1]];
  const int64_t e0 = tile * (int64_t)LT;
  if (e0 >= ntot) return;
  const int64_t e1 = min(e0 + (int64_t)LT, ntot);

  // this thread's kept outputs of a single-round tile stay in registers until the
  // tile's output offset is known
  T o_t[LPT];
  VT o_v[LPT];
  double o_v2[LPT];
  int my_koff = 0;
  unsigned my_kmask = 0;
  bool multi = false;

  int64_t kr = tile_node[tile];
  int64_t rs = e0;
  int kept_run = 0;
  while (rs < e1) {
    // ---- 1. segment table for this round
    int valid = 0;
    {
      const int64_t kk = kr + tid;
      if (tid < MAXSEG && kk < nout) {
        const int64_t s = src[kk];
        const int c = cnt[kk];
        const int64_t b = off[s];
        const int64_t la = off[s + 1] - b;
        const int64_t lb = (c == 2) ? off[s + 2] - off[s + 1] : 0;
        const int64_t ss = max(rs, b), se = min(e1, b + la + lb);
        if (ss < se) {
          valid = 1;
          Seg g;
          g.node = kk;
          g.base = b;
          g.na = la;
          g.nb = lb;
          g.m0 = ss - b;
          g.m1 = se - b;
          g.pass = (c == 1);
          if (g.pass) {
            g.i0 = g.m0; g.j0 = 0; g.i1 = g.m1; g.j1 = 0;
          } else {
            // partial segments only occur at the tile edges, where the partition kernel
            // already found the co-ranks
            g.i0 = g.m0 == 0 ? 0 : tile_i[tile];
            g.j0 = g.m0 - g.i0;
            g.i1 = g.m1 == la + lb ? la : tile_i[tile + 1];
            g.j1 = g.m1 - g.i1;
          }
          g.ia_lo = g.i0 > 0 ? g.i0 - 1 : 0;
          g.jb_lo = g.j0 > 0 ? g.j0 - 1 : 0;
          g.alen = (int)(min(g.i1 + 1, la) - g.ia_lo);
          g.blen = lb > 0 ? (int)(min(g.j1 + 1, lb) - g.jb_lo) : 0;
          g.ga = b + g.ia_lo;
          g.gb = b + la + g.jb_lo;
          if (MOM && !g.pass) {
            const double nA = (double)leaves[s], nB = (double)leaves[s + 1];
            const double n = nA + nB;
            g.wB = nB / n;
            g.wAB = nA * nB / n;
          } else {
            g.wB = g.wAB = 0.0;
          }
          seg[tid] = g;
        }
      }
    }
    const int nseg = __syncthreads_count(valid);
    // window offsets: each window padded out to whole 16-byte granules of the global
    // arrays (exclusive scan of the padded lengths keeps every window granule-aligned)
    int la_p = 0, lb_p = 0;
    if (tid < nseg) {
      const Seg& g = seg[tid];
      la_p = (int)(((g.ga + g.alen + U - 1) & ~(int64_t)(U - 1)) - (g.ga & ~(int64_t)(U - 1)));
      lb_p = g.blen > 0 ? (int)(((g.gb + g.blen + U - 1) & ~(int64_t)(U - 1)) -
                                (g.gb & ~(int64_t)(U - 1)))
                        : 0;
    }
    int woff, wtot;
    woff = block_exclusive_sum<LTH>(la_p + lb_p, scan_ws, &wtot);
    if (tid < nseg) {
      seg[tid].aoff = woff + (int)(seg[tid].ga & (U - 1));
      seg[tid].boff = woff + la_p + (int)(seg[tid].gb & (U - 1));
      seg_pos[tid] = (int)(seg[tid].base + seg[tid].m0 - rs);
    }
    if (tid == 0) {
      const Seg& last = seg[nseg - 1];
      s_round_end = last.base + last.m1;
      s_next_node = kr + nseg;
      seg_pos[nseg] = (int)(s_round_end - rs);
    }
    // ---- 2. stage the input windows with TMA bulk copies (one issuing thread per
    //        segment; whole granules up to the last one, which may end past the array and
    //        is loaded element-wise instead)
    if (tid < nseg) {
      const Seg g = seg[tid];
      fence_proxy_async();
      uint32_t bytes = 0;
      int64_t lo_[2], hi_[2];
      int dst_[2];
      lo_[0] = g.ga & ~(int64_t)(U - 1);
      hi_[0] = (g.ga + g.alen) & ~(int64_t)(U - 1);
      dst_[0] = woff;
      lo_[1] = g.gb & ~(int64_t)(U - 1);
      hi_[1] = g.blen > 0 ? ((g.gb + g.blen) & ~(int64_t)(U - 1)) : lo_[1];
      dst_[1] = woff + la_p;
      for (int w = 0; w < 2; ++w)
        if (hi_[w] > lo_[w])
          bytes += (uint32_t)((hi_[w] - lo_[w]) * (sizeof(T) + sizeof(VT) + (MOM ? 8 : 0)));
      if (bytes) mbar_expect_tx(&s_bar, bytes);
      for (int w = 0; w < 2; ++w) {
        if (hi_[w] > lo_[w]) {
          const uint32_t n = (uint32_t)(hi_[w] - lo_[w]);
          bulk_g2s(s_t + dst_[w], t + lo_[w], n * (uint32_t)sizeof(T), &s_bar);
          bulk_g2s(s_v + dst_[w], v + lo_[w], n * (uint32_t)sizeof(VT), &s_bar);
          if (MOM) bulk_g2s(s_v2 + dst_[w], v2 + lo_[w], n * 8u, &s_bar);
        }
        // the partial last granule, element-wise
        const int64_t e = w == 0 ? g.ga + g.alen : (g.blen > 0 ? g.gb + g.blen : 0);
        for (int64_t x = max(hi_[w], lo_[w]); x < e; ++x) {
          const int d = dst_[w] + (int)(x - lo_[w]);
          s_t[d] = t[x];
          s_v[d] = v[x];
          if (MOM) s_v2[d] = v2[x];
        }
      }
    }
    __syncthreads();  // every expect_tx is registered before the single arrival
    if (tid == 0) mbar_arrive(&s_bar);
    const int64_t re = s_round_end;
    if (rs == e0 && re < e1) multi = true;  // the tile needs more than one round
    mbar_wait(&s_bar, bar_phase);
    bar_phase ^= 1u;
    __syncthreads();  // element-wise tails visible
    // ---- 3. walk LPT positions per thread, once: values + keep flags into registers
    const int p0 = tid * LPT;  // round-relative
    const int rlen = (int)(re - rs);
    unsigned kmask = 0, nsmask = 0;
    if (p0 < rlen) {
      int sg;
      {
        int lo = 0, hi = nseg - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (seg_pos[mid] <= p0) lo = mid;
          else hi = mid - 1;
        }
        sg = lo;
      }
      Seg g = seg[sg];  // register copy of the current segment
      // 32-bit walk state; shared-memory base pointers shifted so that A element x of the
      // node is at pa_t[x] (only the staged window is ever dereferenced)
      int m = 0, i = 0, j = 0;
      const T* pa_t;
      const T* pb_t;
      const VT* pa_v;
      const VT* pb_v;
      const double* pa_2;
      const double* pb_2;
      auto bind = [&]() {
        pa_t = s_t + g.aoff - (int)g.ia_lo;
        pb_t = s_t + g.boff - (int)g.jb_lo;
        pa_v = s_v + g.aoff - (int)g.ia_lo;
        pb_v = s_v + g.boff - (int)g.jb_lo;
        pa_2 = s_v2 + g.aoff - (int)g.ia_lo;
        pb_2 = s_v2 + g.boff - (int)g.jb_lo;
      };
      bind();
      VT pv = VT(0);
      double pv2 = 0.0;
      auto TA = [&](int x) { return pa_t[x]; };
      auto TB = [&](int x) { return pb_t[x]; };
      auto VA = [&](int x) { return pa_v[x]; };
      auto VB = [&](int x) { return pb_v[x]; };
      auto V2A = [&](int x) { return pa_2[x]; };
      auto V2B = [&](int x) { return pb_2[x]; };
      auto comb = [&](int ia, int ib, VT& ov, double& ov2) {
        if (MOM) {
          const double d = (double)VB(ib) - (double)VA(ia);
          ov = (VT)((double)VA(ia) + d * g.wB);
          ov2 = (V2A(ia) + V2B(ib)) + d * d * g.wAB;
        } else {
          ov = to_t<VT>(vop<K>((double)VA(ia), (double)VB(ib)));
          ov2 = 0.0;
        }
      };
      auto start = [&](int mm) {
        m = mm;
        if (g.pass) {
          i = mm;
          j = 0;
          return;
        }
        // co-ranks are monotone in m: i in [i0, i1], j = m - i in [j0, j1]
        int lo = max((int)g.i0, mm - (int)g.j1), hi = min((int)g.i1, mm - (int)g.j0);
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (TA(mid) <= TB(mm - mid - 1)) lo = mid + 1;
          else hi = mid;
        }
        i = lo;
        j = mm - lo;
        if (mm > 0) {
          const T tp = (j > 0 && TB(j - 1) > TA(i - 1)) ? TB(j - 1) : TA(i - 1);
          const int jt = j + ((j < (int)g.nb && TB(j) == tp) ? 1 : 0) - 1;
          comb(i - 1, jt, pv, pv2);
        }
      };
      // branch-free merge state for merged segments: next A / B breakpoints in registers
      // (+inf past the end), the last A breakpoint taken (duplicate test for B)
      const T TINF = (T)INFINITY;
      T tai = TINF, tbj = TINF, taprev = (T)-1;
      auto load_state = [&]() {
        if (g.pass) return;
        tai = i < (int)g.na ? TA(i) : TINF;
        tbj = j < (int)g.nb ? TB(j) : TINF;
        taprev = i > 0 ? TA(i - 1) : (T)-1;
      };
      start((int)g.m0 + (p0 - seg_pos[sg]));
      load_state();
#pragma unroll
      for (int q = 0; q < LPT; ++q) {
        const int p = p0 + q;
        if (p < rlen) {
          if (sg + 1 < nseg && p >= seg_pos[sg + 1]) {
            ++sg;
            g = seg[sg];
            bind();
            start((int)g.m0);
            load_state();
          }
          T tt;
          VT val = pv;
          double val2 = pv2;
          int kp;
          if (m == 0) nsmask |= 1u << q;  // node start: first candidate, always kept
          if (g.pass) {
            tt = TA(i);
            val = VA(i);
            if (MOM) val2 = V2A(i);
            kp = 1;
            ++i;
          } else {
            const bool takeA = tai <= tbj;  // A first on ties (stable merge)
            tt = takeA ? tai : tbj;
            const bool dup = !takeA && (taprev == tt);
            const int ia = takeA ? i : i - 1;
            const int ib = takeA ? j - 1 + (tbj == tt ? 1 : 0) : j;
            comb(ia, ib, val, val2);
            kp = !dup && ((m == 0) || (val != pv) || (MOM && val2 != pv2));
            if (!dup) {
              pv = val;
              pv2 = val2;
            }
            if (takeA) taprev = tai;
            i += takeA ? 1 : 0;
            j += takeA ? 0 : 1;
            // reload only the advanced cursor's next breakpoint (one selected load)
            const bool inA = takeA ? (i < (int)g.na) : (j < (int)g.nb);
            const T nxt = inA ? (takeA ? TA(i) : TB(j)) : TINF;
            tai = takeA ? nxt : tai;
            tbj = takeA ? tbj : nxt;
          }
          ++m;
          o_t[q] = tt;
          o_v[q] = val;
          o_v2[q] = val2;
          if (kp) {
            kmask |= 1u << q;
            if (!MOM && !isfinite((double)val)) atomicOr(status, 1);
          }
        }
      }
    }
    const int nk = __popc(kmask);
    int koff, ktot;
    koff = block_exclusive_sum<LTH>(nk, scan_ws, &ktot);
    // node starts of this round: tile-local output index now, the tile's offset is added
    // by k_fix_offsets after the level (tile_excl)
    if (nsmask) {
      int r = 0;
#pragma unroll
      for (int q = 0; q < LPT; ++q) {
        if ((kmask >> q) & 1u) {
          if ((nsmask >> q) & 1u) {
            const int p = p0 + q;
            int lo = 0, hi = nseg - 1;
            while (lo < hi) {
              const int mid = (lo + hi + 1) >> 1;
              if (seg_pos[mid] <= p) lo = mid;
              else hi = mid - 1;
            }
            off_out[seg[lo].node] = kept_run + koff + r;
          }
          ++r;
        }
      }
    }
    if (multi) {  // park this round's kept points in the tile's scratch region
      int r = 0;
#pragma unroll
      for (int q = 0; q < LPT; ++q) {
        if ((kmask >> q) & 1u) {
          const int64_t x = e0 + kept_run + koff + r;
          x_t[x] = o_t[q];
          x_v[x] = o_v[q];
          if (MOM) x_v2[x] = o_v2[q];
          ++r;
        }
      }
    } else {
      my_koff = koff;
      my_kmask = kmask;
    }
    kept_run += ktot;
    rs = re;
    kr = s_next_node;
    __syncthreads();  // shared tables are rebuilt next round
  }
  // ---- 4. decoupled look-back: the tile's output offset.  One warp inspects 32
  //        predecessors per step (one L2 round trip), sums their aggregates back to the
  //        nearest inclusive prefix, and publishes this tile's inclusive prefix.
  if (tid < 32) {
    constexpr unsigned long long AGG = 1ull << 62, PRE = 2ull << 62, VAL = (1ull << 62) - 1;
    volatile unsigned long long* st = tile_status;
    const int lane = tid;
    unsigned long long excl = 0;
    if (tile == 0) {
      if (lane == 0) st[0] = PRE | (unsigned long long)kept_run;
    } else {
      if (lane == 0) st[tile] = AGG | (unsigned long long)kept_run;
      for (int64_t base = tile - 1;; base -= 32) {
        const int64_t pt = base - lane;
        unsigned long long w = pt >= 0 ? st[pt] : PRE;  // before tile 0: prefix 0
        while (__any_sync(0xffffffffu, (w >> 62) == 0)) {
          if ((w >> 62) == 0) w = st[pt];  // predecessor not published yet: spin
        }
        const unsigned pre = __ballot_sync(0xffffffffu, (w >> 62) == 2);
        const int first = pre ? __ffs(pre) - 1 : 32;  // nearest inclusive prefix
        unsigned long long val = lane <= first ? (w & VAL) : 0ull;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        excl += val;
        if (pre) break;
      }
      if (lane == 0) st[tile] = PRE | (excl + (unsigned long long)kept_run);
    }
    if (lane == 0) s_excl = (int64_t)excl;
  }
  __syncthreads();
  const int64_t out_base = s_excl;
  // ---- 5. write the kept points: through the (now free) window buffers so the global
  //         stores are coalesced rows instead of per-thread strided runs
  if (!multi) {
    int r = 0;
#pragma unroll
    for (int q = 0; q < LPT; ++q) {
      if ((my_kmask >> q) & 1u) {
        const int x = my_koff + r;
        const int y = x + x / LPT;  // one pad slot per LPT: few bank conflicts
        s_t[y] = o_t[q];
        s_v[y] = o_v[q];
        if (MOM) s_v2[y] = o_v2[q];
        ++r;
      }
    }
    __syncthreads();
    for (int x = tid; x < kept_run; x += LTH) {
      const int y = x + x / LPT;
      t_out[out_base + x] = s_t[y];
      v_out[out_base + x] = s_v[y];
      if (MOM) v2_out[out_base + x] = s_v2[y];
    }
  } else {
    for (int x = tid; x < kept_run; x += LTH) {
      t_out[out_base + x] = x_t[e0 + x];
      v_out[out_base + x] = x_v[e0 + x];
      if (MOM) v2_out[out_base + x] = x_v2[e0 + x];
    }
  }
  if (tid == 0) {
    tile_excl[tile] = out_base;
    if (e1 == ntot) off_out[nout] = out_base + kept_run;
  }
}

// Output node offsets: node k starts in the tile holding its first candidate
// (off[src[k]]); the level kernel stored the tile-local index, add the tile's offset.
__global__ void k_fix_offsets(const int64_t* __restrict__ off, const int64_t* __restrict__ src,
                              int64_t nout, const int64_t* __restrict__ tile_excl,
                              int64_t* __restrict__ off_out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nout;
       k += (int64_t)gridDim.x * blockDim.x)
    off_out[k] += tile_excl[off[src[k]] / LT];
}

// Non-compacting level (K5m): the same merge as k_level_tiled, but every candidate is
// kept at its own input position -- no keep flags, no scan, no look-back, node offsets
// unchanged.  Used above the first level when breakpoints are (nearly) distinct, where
// compaction would drop almost nothing.  A breakpoint time present in both children
// yields two consecutive points with the same time: the first is a zero-width piece
// (its value combines one child's jump with the other child's previous value, which the
// reference never forms), the second carries the exact reference value.  Survivors only
// ever combine survivors, so every last-of-its-time point equals the reference tree value
// bit for bit; the finalisation (k_scale_flag / k_std_flag with times) drops zero-width
// pieces and then minimises, which is the reference's result (intermediate emission
// never changes values, only which redundant points exist).
template <typename T, int K, int MT>
__global__ void __launch_bounds__(MT, (K == K_MOM ? 3 : 4) * 256 / MT)
    k_merge_level(const T* __restrict__ t, const void* __restrict__ v_,
                  const double* __restrict__ v2, const int64_t* __restrict__ off,
                  const int64_t* __restrict__ src, const int32_t* __restrict__ cnt,
                  const int64_t* __restrict__ leaves, int64_t nout,
                  const int64_t* __restrict__ tile_node, const int64_t* __restrict__ tile_i,
                  T* __restrict__ t_out, void* __restrict__ v_out_, double* __restrict__ v2_out) {
  using VT = typename std::conditional<K == K_MOM, double, T>::type;
  const VT* __restrict__ v = reinterpret_cast<const VT*>(v_);
  VT* __restrict__ v_out = reinterpret_cast<VT*>(v_out_);
  constexpr bool MOM = (K == K_MOM);
  constexpr int MLT = MT * LPT;  // candidate positions per tile
  constexpr int WCAP = MLT + (4 + 4 * (16 / (int)sizeof(T) - 1)) * MAXSEG;
  constexpr int U = 16 / (int)sizeof(T);

  __shared__ Seg seg[MAXSEG];
  __shared__ int seg_pos[MAXSEG + 1];
  extern __shared__ __align__(16) unsigned char dyn[];
  VT* s_v = reinterpret_cast<VT*>(dyn);
  double* s_v2 = reinterpret_cast<double*>(dyn + WCAP * sizeof(VT));
  T* s_t = reinterpret_cast<T*>(dyn + WCAP * sizeof(VT) + (MOM ? WCAP * sizeof(double) : 0));
  __shared__ uint64_t s_bar;
  __shared__ int64_t s_next_node, s_round_end;
  __shared__ int scan_ws[MT / 32];

  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    fence_mbar_init();
  }
  uint32_t bar_phase = 0;
  __syncthreads();
  const int64_t tile = blockIdx.x;
  const int64_t ntot = off[src[nout - 1] + cnt[nout - 1]];
  const int64_t e0 = tile * (int64_t)MLT;
  if (e0 >= ntot) return;
  const int64_t e1 = min(e0 + (int64_t)MLT, ntot);
  int64_t kr = tile_node[tile];
  int64_t rs = e0;
  while (rs < e1) {
    int valid = 0;
    {
      const int64_t kk = kr + tid;
      if (tid < MAXSEG && kk < nout) {
        const int64_t s = src[kk];
        const int c = cnt[kk];
        const int64_t b = off[s];
        const int64_t la = off[s + 1] - b;
        const int64_t lb = (c == 2) ? off[s + 2] - off[s + 1] : 0;
        const int64_t ss = max(rs, b), se = min(e1, b + la + lb);
        if (ss < se) {
          valid = 1;
          Seg g;
          g.node = kk;
          g.base = b;
          g.na = la;
          g.nb = lb;
          g.m0 = ss - b;
          g.m1 = se - b;
          g.pass = (c == 1);
          if (g.pass) {
            g.i0 = g.m0; g.j0 = 0; g.i1 = g.m1; g.j1 = 0;
          } else {
            g.i0 = g.m0 == 0 ? 0 : tile_i[tile];
            g.j0 = g.m0 - g.i0;
            g.i1 = g.m1 == la + lb ? la : tile_i[tile + 1];
            g.j1 = g.m1 - g.i1;
          }
          g.ia_lo = g.i0 > 0 ? g.i0 - 1 : 0;
          g.jb_lo = g.j0 > 0 ? g.j0 - 1 : 0;
          g.alen = (int)(min(g.i1 + 1, la) - g.ia_lo);
          g.blen = lb > 0 ? (int)(min(g.j1 + 1, lb) - g.jb_lo) : 0;
          g.ga = b + g.ia_lo;
          g.gb = b + la + g.jb_lo;
          if (MOM && !g.pass) {
            const double nA = (double)leaves[s], nB = (double)leaves[s + 1];
            const double n = nA + nB;
            g.wB = nB / n;
            g.wAB = nA * nB / n;
          } else {
            g.wB = g.wAB = 0.0;
          }
          seg[tid] = g;
        }
      }
    }
    const int nseg = __syncthreads_count(valid);
    int la_p = 0, lb_p = 0;
    if (tid < nseg) {
      const Seg& g = seg[tid];
      la_p = (int)(((g.ga + g.alen + U - 1) & ~(int64_t)(U - 1)) - (g.ga & ~(int64_t)(U - 1)));
      lb_p = g.blen > 0 ? (int)(((g.gb + g.blen + U - 1) & ~(int64_t)(U - 1)) -
                                (g.gb & ~(int64_t)(U - 1)))
                        : 0;
    }
    int woff, wtot;
    woff = block_exclusive_sum<MT>(la_p + lb_p, scan_ws, &wtot);
    if (tid < nseg) {
      seg[tid].aoff = woff + (int)(seg[tid].ga & (U - 1));
      seg[tid].boff = woff + la_p + (int)(seg[tid].gb & (U - 1));
      seg_pos[tid] = (int)(seg[tid].base + seg[tid].m0 - rs);
    }
    if (tid == 0) {
      const Seg& last = seg[nseg - 1];
      s_round_end = last.base + last.m1;
      s_next_node = kr + nseg;
      seg_pos[nseg] = (int)(s_round_end - rs);
    }
    if (tid < nseg) {
      const Seg g = seg[tid];
      fence_proxy_async();
      uint32_t bytes = 0;
      int64_t lo_[2], hi_[2];
      int dst_[2];
      lo_[0] = g.ga & ~(int64_t)(U - 1);
      hi_[0] = (g.ga + g.alen) & ~(int64_t)(U - 1);
      dst_[0] = woff;
      lo_[1] = g.gb & ~(int64_t)(U - 1);
      hi_[1] = g.blen > 0 ? ((g.gb + g.blen) & ~(int64_t)(U - 1)) : lo_[1];
      dst_[1] = woff + la_p;
      for (int w = 0; w < 2; ++w)
        if (hi_[w] > lo_[w])
          bytes += (uint32_t)((hi_[w] - lo_[w]) * (sizeof(T) + sizeof(VT) + (MOM ? 8 : 0)));
      if (bytes) mbar_expect_tx(&s_bar, bytes);
      for (int w = 0; w < 2; ++w) {
        if (hi_[w] > lo_[w]) {
          const uint32_t n = (uint32_t)(hi_[w] - lo_[w]);
          bulk_g2s(s_t + dst_[w], t + lo_[w], n * (uint32_t)sizeof(T), &s_bar);
          bulk_g2s(s_v + dst_[w], v + lo_[w], n * (uint32_t)sizeof(VT), &s_bar);
          if (MOM) bulk_g2s(s_v2 + dst_[w], v2 + lo_[w], n * 8u, &s_bar);
        }
        const int64_t e = w == 0 ? g.ga + g.alen : (g.blen > 0 ? g.gb + g.blen : 0);
        for (int64_t x = max(hi_[w], lo_[w]); x < e; ++x) {
          const int d = dst_[w] + (int)(x - lo_[w]);
          s_t[d] = t[x];
          s_v[d] = v[x];
          if (MOM) s_v2[d] = v2[x];
        }
      }
    }
    __syncthreads();
    if (tid == 0) mbar_arrive(&s_bar);
    const int64_t re = s_round_end;
    mbar_wait(&s_bar, bar_phase);
    bar_phase ^= 1u;
    __syncthreads();
    // ---- walk: every candidate lands at its own position rs + p; values are collected in
    //      registers and written out through shared memory as coalesced rows (thread-
    //      strided global stores made the L1 the bottleneck of this kernel)
    const int p0 = tid * LPT;
    const int rlen = (int)(re - rs);
    T o_t[LPT];
    VT o_v[LPT];
    double o_v2[LPT];
    if (p0 < rlen) {
      int sg;
      {
        int lo = 0, hi = nseg - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (seg_pos[mid] <= p0) lo = mid;
          else hi = mid - 1;
        }
        sg = lo;
      }
      Seg g = seg[sg];
      int i = 0, j = 0;
      const T* pa_t;
      const T* pb_t;
      const VT* pa_v;
      const VT* pb_v;
      const double* pa_2;
      const double* pb_2;
      auto bind = [&]() {
        pa_t = s_t + g.aoff - (int)g.ia_lo;
        pb_t = s_t + g.boff - (int)g.jb_lo;
        pa_v = s_v + g.aoff - (int)g.ia_lo;
        pb_v = s_v + g.boff - (int)g.jb_lo;
        pa_2 = s_v2 + g.aoff - (int)g.ia_lo;
        pb_2 = s_v2 + g.boff - (int)g.jb_lo;
      };
      bind();
      const T TINF = (T)INFINITY;
      T tai = TINF, tbj = TINF;
      auto start = [&](int mm) {
        if (g.pass) {
          i = mm;
          j = 0;
          return;
        }
        int lo = max((int)g.i0, mm - (int)g.j1), hi = min((int)g.i1, mm - (int)g.j0);
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (pa_t[mid] <= pb_t[mm - mid - 1]) lo = mid + 1;
          else hi = mid;
        }
        i = lo;
        j = mm - lo;
        tai = i < (int)g.na ? pa_t[i] : TINF;
        tbj = j < (int)g.nb ? pb_t[j] : TINF;
      };
      start((int)g.m0 + (p0 - seg_pos[sg]));
#pragma unroll
      for (int q = 0; q < LPT; ++q) {
        const int p = p0 + q;
        if (p < rlen) {
          if (sg + 1 < nseg && p >= seg_pos[sg + 1]) {
            ++sg;
            g = seg[sg];
            bind();
            start((int)g.m0);
          }
          T tt;
          VT val;
          double val2 = 0.0;
          if (g.pass) {
            tt = pa_t[i];
            val = pa_v[i];
            if (MOM) val2 = pa_2[i];
            ++i;
          } else {
            const bool takeA = tai <= tbj;  // A first on ties (stable merge)
            tt = takeA ? tai : tbj;
            const int ia = takeA ? i : i - 1;
            int ib = takeA ? j - 1 : j;
            ib = ib < 0 ? 0 : ib;  // a t = 0 zero-width piece before B's first point
            if (MOM) {
              const double d = (double)pb_v[ib] - (double)pa_v[ia];
              val = (VT)((double)pa_v[ia] + d * g.wB);
              val2 = (pa_2[ia] + pb_2[ib]) + d * d * g.wAB;
            } else {
              val = to_t<VT>(vop<K>((double)pa_v[ia], (double)pb_v[ib]));
            }
            i += takeA ? 1 : 0;
            j += takeA ? 0 : 1;
            const bool inA = takeA ? (i < (int)g.na) : (j < (int)g.nb);
            const T nxt = inA ? (takeA ? pa_t[i] : pb_t[j]) : TINF;
            tai = takeA ? nxt : tai;
            tbj = takeA ? tbj : nxt;
          }
          o_t[q] = tt;
          o_v[q] = val;
          if (MOM) o_v2[q] = val2;
        }
      }
    }
    __syncthreads();  // the staged windows are free: reuse them for the output rows
    {
      // element p at p + p / LPT (one pad slot per thread: 2-way bank conflicts at most)
#pragma unroll
      for (int q = 0; q < LPT; ++q) {
        if (p0 + q < rlen) {
          const int x = p0 + q + tid;
          s_t[x] = o_t[q];
          s_v[x] = o_v[q];
          if (MOM) s_v2[x] = o_v2[q];
        }
      }
    }
    __syncthreads();
    for (int x = tid; x < rlen; x += MT) {
      const int y = x + x / LPT;
      t_out[rs + x] = s_t[y];
      v_out[rs + x] = s_v[y];
      if (MOM) v2_out[rs + x] = s_v2[y];
    }
    rs = re;
    kr = s_next_node;
    __syncthreads();
  }
}

// Output node offsets of a non-compacting level: node k starts where its first child did.
__global__ void k_merge_offsets(const int64_t* __restrict__ off, const int64_t* __restrict__ src,
                                const int32_t* __restrict__ cnt, int64_t nout,
                                int64_t* __restrict__ off_out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= nout;
       k += (int64_t)gridDim.x * blockDim.x)
    off_out[k] = k < nout ? off[src[k]] : off[src[nout - 1] + cnt[nout - 1]];
}

// Merge-path partition: for every tile start (and the end of the last tile) the output
// node containing it (largest k with off[src[k]] <= e) and the co-rank (A elements among
// the node's first m candidates).
template <typename T>
__global__ void k_tile_part(const T* __restrict__ t, const int64_t* __restrict__ off,
                            const int64_t* __restrict__ src, const int32_t* __restrict__ cnt,
                            int64_t nout, int64_t ntot, int64_t ntiles,
                            int64_t* __restrict__ tile_node, int64_t* __restrict__ tile_i,
                            int64_t lt = LT) {
  ntot = off[src[nout - 1] + cnt[nout - 1]];  // live point count (ntot: upper bound)
  for (int64_t tl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; tl <= ntiles;
       tl += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = min(tl * lt, ntot);
    int64_t lo = 0, hi = nout - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (off[src[mid]] <= e) lo = mid;
      else hi = mid - 1;
    }
    const int64_t s = src[lo];
    const int64_t b = off[s];
    const int64_t la = off[s + 1] - b;
    const int64_t m = e - b;
    int64_t i;
    if (cnt[lo] == 1) {
      i = m;
    } else {
      const int64_t lb = off[s + 2] - off[s + 1];
      i = (m >= la + lb) ? la : corank_g(t + b, la, t + b + la, lb, m);
    }
    tile_node[tl] = lo;
    tile_i[tl] = i;
  }
}

}  // namespace lvl
}  // namespace pcfb

using namespace pcfb;
using namespace pcfb::lvl;

extern "C" {

int pcf_tree_level_workspace(int64_t ntot, int64_t* bytes) {
  // tile_node, tile_i, tile_status (+counter), tile_excl: ntiles+1 words each; scratch for
  // multi-round tiles: t, v, v2 (8 bytes each) per candidate
  const int64_t ntiles = (ntot + LT - 1) / LT;
  *bytes = (int64_t)(4 * 8 * (ntiles + 2) + 64 + 3 * 8 * (ntot > 0 ? ntot : 1) + 256);
  return PCF_OK;
}

int pcf_tree_level(int kind, int is_f32, const void* t_dev, const void* v_dev,
                   const double* v2_dev, const int64_t* off_dev, const int64_t* src_dev,
                   const int32_t* cnt_dev, const int64_t* leaves_dev, int64_t nout,
                   int64_t ntot, void* t_out_dev, void* v_out_dev, double* v2_out_dev,
                   int64_t* off_out_dev, void* ws_dev, int64_t ws_bytes, int32_t* status_dev,
                   void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (nout <= 0) return PCF_OK;
  if (kind < 0 || kind > 4 || !t_dev || !v_dev || !off_dev || !src_dev || !cnt_dev ||
      !t_out_dev || !v_out_dev || !off_out_dev || !ws_dev || !status_dev ||
      (kind == K_MOM && (!v2_dev || !v2_out_dev || !leaves_dev))) {
    set_error("pcf_tree_level: bad arguments");
    return PCF_ERR_ARG;
  }
  if (ntot <= 0) {
    const cudaError_t e0 = cudaMemsetAsync(off_out_dev, 0, (nout + 1) * sizeof(int64_t), s);
    if (e0 != cudaSuccess) {
      set_error("pcf_tree_level: %s", cudaGetErrorString(e0));
      return PCF_ERR_CUDA;
    }
    return PCF_OK;
  }
  const int64_t ntiles = (ntot + LT - 1) / LT;
  int64_t need = 0;
  pcf_tree_level_workspace(ntot, &need);
  if (ws_bytes < need) {
    set_error("pcf_tree_level: workspace %lld < %lld bytes", (long long)ws_bytes,
              (long long)need);
    return PCF_ERR_ARG;
  }
  int64_t* tile_node = (int64_t*)ws_dev;
  int64_t* tile_i = tile_node + (ntiles + 1);
  unsigned long long* tile_status = (unsigned long long*)(tile_i + (ntiles + 1));
  int* tile_counter = (int*)(tile_status + (ntiles + 1));
  int64_t* tile_excl = (int64_t*)(tile_status + (ntiles + 2));
  char* xbase = (char*)(tile_excl + (ntiles + 2));
  xbase = (char*)(((uintptr_t)xbase + 255) & ~(uintptr_t)255);
  void* x_t = xbase;
  void* x_v = xbase + 8 * ntot;
  double* x_v2 = (double*)(xbase + 16 * ntot);
  {
    const cudaError_t e0 = cudaMemsetAsync(tile_status, 0, (ntiles + 1) * 8 + 16, s);
    if (e0 != cudaSuccess) {
      set_error("pcf_tree_level: %s", cudaGetErrorString(e0));
      return PCF_ERR_CUDA;
    }
  }
  const int pg = (int)((ntiles + 1 + 255) / 256);
  const unsigned grid = (unsigned)ntiles;
#define PCF_TL(T, K)                                                                          \
  do {                                                                                        \
    typedef typename std::conditional<K == K_MOM, double, T>::type VT_;                      \
    const int dsm = wcap<T>() * (int)(sizeof(VT_) + sizeof(T) + (K == K_MOM ? sizeof(double) : 0)); \
    cudaFuncSetAttribute(k_level_tiled<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                         dsm);                                                                \
    k_level_tiled<T, K><<<grid, LTH, dsm, s>>>(                                               \
        (const T*)t_dev, v_dev, v2_dev, off_dev, src_dev, cnt_dev, leaves_dev, nout, ntot,   \
        tile_node, tile_i, tile_counter, tile_status, (T*)t_out_dev, v_out_dev, v2_out_dev,   \
        off_out_dev, status_dev, tile_excl, (T*)x_t, x_v, x_v2);                              \
  } while (0)
#define PCF_TL_BOTH(T, K)                                                                     \
  do {                                                                                        \
    k_tile_part<T><<<pg, 256, 0, s>>>((const T*)t_dev, off_dev, src_dev, cnt_dev, nout, ntot, \
                                      ntiles, tile_node, tile_i);                             \
    PCF_TL(T, K);                                                                             \
    k_fix_offsets<<<(unsigned)((nout + 255) / 256 < 4096 ? (nout + 255) / 256 : 4096), 256,   \
                    0, s>>>(off_dev, src_dev, nout, tile_excl, off_out_dev);                  \
  } while (0)
  if (is_f32) {
    switch (kind) {
      case K_ADD: PCF_TL_BOTH(float, K_ADD); break;
      case K_MAX: PCF_TL_BOTH(float, K_MAX); break;
      case K_MIN: PCF_TL_BOTH(float, K_MIN); break;
      case K_MUL: PCF_TL_BOTH(float, K_MUL); break;
      default: PCF_TL_BOTH(float, K_MOM); break;
    }
  } else {
    switch (kind) {
      case K_ADD: PCF_TL_BOTH(double, K_ADD); break;
      case K_MAX: PCF_TL_BOTH(double, K_MAX); break;
      case K_MIN: PCF_TL_BOTH(double, K_MIN); break;
      case K_MUL: PCF_TL_BOTH(double, K_MUL); break;
      default: PCF_TL_BOTH(double, K_MOM); break;
    }
  }
#undef PCF_TL_BOTH
#undef PCF_TL
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("pcf_tree_level: %s", cudaGetErrorString(e));
    return PCF_ERR_CUDA;
  }
  return PCF_OK;
}

int pcf_tree_merge_level(int kind, int is_f32, const void* t_dev, const void* v_dev,
                         const double* v2_dev, const int64_t* off_dev, const int64_t* src_dev,
                         const int32_t* cnt_dev, const int64_t* leaves_dev, int64_t nout,
                         int64_t ntot, void* t_out_dev, void* v_out_dev, double* v2_out_dev,
                         int64_t* off_out_dev, void* ws_dev, int64_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (nout <= 0) return PCF_OK;
  if (kind < 0 || kind > 4 || !t_dev || !v_dev || !off_dev || !src_dev || !cnt_dev ||
      !t_out_dev || !v_out_dev || !off_out_dev || !ws_dev ||
      (kind == K_MOM && (!v2_dev || !v2_out_dev || !leaves_dev))) {
    set_error("pcf_tree_merge_level: bad arguments");
    return PCF_ERR_ARG;
  }
  const int og = (int)((nout + 1 + 255) / 256 < 4096 ? (nout + 1 + 255) / 256 : 4096);
  k_merge_offsets<<<og, 256, 0, s>>>(off_dev, src_dev, cnt_dev, nout, off_out_dev);
  if (ntot <= 0) return PCF_OK;
  constexpr int MT = 256;  // threads per merge tile (MT * LPT positions; 128 and 512 measured slower)
  constexpr int64_t MLT = (int64_t)MT * LPT;
  const int64_t ntiles = (ntot + MLT - 1) / MLT;
  int64_t need = 0;
  pcf_tree_level_workspace(ntot, &need);
  if (ws_bytes < need) {
    set_error("pcf_tree_merge_level: workspace %lld < %lld bytes", (long long)ws_bytes,
              (long long)need);
    return PCF_ERR_ARG;
  }
  int64_t* tile_node = (int64_t*)ws_dev;
  int64_t* tile_i = tile_node + (ntiles + 1);
  const int pg = (int)((ntiles + 1 + 255) / 256);
  const unsigned grid = (unsigned)ntiles;
#define PCF_ML(T, K)                                                                          \
  do {                                                                                        \
    typedef typename std::conditional<K == K_MOM, double, T>::type VT_;                      \
    const int wc = (int)MLT + (4 + 4 * (16 / (int)sizeof(T) - 1)) * MAXSEG;                 \
    const int dsm = wc * (int)(sizeof(VT_) + sizeof(T) + (K == K_MOM ? sizeof(double) : 0)); \
    k_tile_part<T><<<pg, 256, 0, s>>>((const T*)t_dev, off_dev, src_dev, cnt_dev, nout, ntot, \
                                      ntiles, tile_node, tile_i, MLT);                        \
    cudaFuncSetAttribute(k_merge_level<T, K, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         dsm);                                                                \
    k_merge_level<T, K, MT><<<grid, MT, dsm, s>>>((const T*)t_dev, v_dev, v2_dev, off_dev,    \
                                               src_dev, cnt_dev, leaves_dev, nout, tile_node, \
                                               tile_i, (T*)t_out_dev, v_out_dev, v2_out_dev); \
  } while (0)
  if (is_f32) {
    switch (kind) {
      case K_ADD: PCF_ML(float, K_ADD); break;
      case K_MAX: PCF_ML(float, K_MAX); break;
      case K_MIN: PCF_ML(float, K_MIN); break;
      case K_MUL: PCF_ML(float, K_MUL); break;
      default: PCF_ML(float, K_MOM); break;
    }
  } else {
    switch (kind) {
      case K_ADD: PCF_ML(double, K_ADD); break;
      case K_MAX: PCF_ML(double, K_MAX); break;
      case K_MIN: PCF_ML(double, K_MIN); break;
      case K_MUL: PCF_ML(double, K_MUL); break;
      default: PCF_ML(double, K_MOM); break;
    }
  }
#undef PCF_ML
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("pcf_tree_merge_level: %s", cudaGetErrorString(e));
    return PCF_ERR_CUDA;
  }
  return PCF_OK;
}


}  // extern "C"
