// Tiled reduction-tree level (K5 / K7, v2): one CTA per tile of LT candidate positions.
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
//   3. each thread walks LPT consecutive positions from shared memory, producing the
//      combined value and reduce_pair's keep flag (value changed w.r.t. the previous
//      cell; duplicate breakpoints dropped; passthrough nodes kept verbatim);
//   4. block scan of the keep flags.
//
// Pass 1 only counts kept points per tile; a device scan of the tile counts gives every
// tile its output offset; pass 2 recomputes the tile (inputs are read twice, nothing
// else round-trips through HBM) and writes the kept points plus the output node offsets.
// HBM traffic per level ~ 3 x 16 B per point for float64 (read, read, write).
#define CCCL_IGNORE_DEPRECATED_API 1
#include <cub/cub.cuh>
#include "pcf_common.cuh"
#include "pcf_internal.h"

namespace pcfb {
namespace lvl {

constexpr int LTH = 256;         // threads per tile CTA
constexpr int LPT = 8;           // positions per thread
constexpr int LT = LTH * LPT;    // candidate positions per tile
constexpr int MAXSEG = 64;       // node segments per round
constexpr int WCAP = LT + 4 * MAXSEG;  // staged elements per round (both windows)

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

template <typename T, int K, bool WRITE>
__global__ void __launch_bounds__(LTH)
    k_level_tiled(const T* __restrict__ t, const void* __restrict__ v_,
                  const double* __restrict__ v2, const int64_t* __restrict__ off,
                  const int64_t* __restrict__ src, const int32_t* __restrict__ cnt,
                  const int64_t* __restrict__ leaves, int64_t nout, int64_t ntot,
                  const int64_t* __restrict__ tile_node, const int64_t* __restrict__ tile_i,
                  int* __restrict__ tile_counter, unsigned long long* __restrict__ tile_status,
                  T* __restrict__ t_out, void* __restrict__ v_out_, double* __restrict__ v2_out,
                  int64_t* __restrict__ off_out, int32_t* __restrict__ status) {
  using VT = typename std::conditional<K == K_MOM, double, T>::type;
  const VT* __restrict__ v = reinterpret_cast<const VT*>(v_);
  VT* __restrict__ v_out = reinterpret_cast<VT*>(v_out_);
  constexpr bool MOM = (K == K_MOM);

  __shared__ Seg seg[MAXSEG];
  __shared__ int seg_pos[MAXSEG + 1];  // tile-relative candidate start of each segment
  extern __shared__ __align__(16) unsigned char dyn[];
  VT* s_v = reinterpret_cast<VT*>(dyn);                          // [WCAP]
  double* s_v2 = reinterpret_cast<double*>(dyn + WCAP * sizeof(VT));  // [WCAP] (moments)
  T* s_t = reinterpret_cast<T*>(dyn + WCAP * sizeof(VT) + (MOM ? WCAP * sizeof(double) : 0));
  __shared__ int64_t s_next_node, s_round_end, s_tile, s_excl;
  typedef cub::BlockScan<int, LTH> Scan;
  __shared__ typename Scan::TempStorage scan_tmp;

  const int tid = threadIdx.x;
  // Tiles are taken in order from an atomic counter, so every tile's predecessors are
  // running or done -- the decoupled look-back below cannot wait on an unscheduled CTA.
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1);
  __syncthreads();
  const int64_t tile = s_tile;
  // `ntot` is a host-side upper bound (the previous level's size); the live point count
  // is the end of the last output node's input range.  Tiles past it are empty.
  ntot = off[src[nout - 1] + cnt[nout - 1]];
  const int64_t e0 = tile * (int64_t)LT;
  if (e0 >= ntot) return;
  const int64_t e1 = min(e0 + (int64_t)LT, ntot);
  int64_t kept_total = 0;
  int koff_saved = 0, rounds = 0, nseg_saved = 0;
  bool single_round = false;

  // One tile = count pass (stage + walk), look-back for the tile's output offset, emit
  // pass (re-stage -- the tile's inputs are still in L2 -- and walk again).
  for (int emit = 0; emit < 2; ++emit) {
  if (emit) {
    if (tid == 0) {
      unsigned long long excl = 0;
      constexpr unsigned long long AGG = 1ull << 62, PRE = 2ull << 62, VAL = (1ull << 62) - 1;
      volatile unsigned long long* st = tile_status;
      if (tile == 0) {
        st[0] = PRE | (unsigned long long)kept_total;
      } else {
        st[tile] = AGG | (unsigned long long)kept_total;
        for (int64_t pt = tile - 1; pt >= 0;) {
          const unsigned long long w = st[pt];
          if ((w >> 62) == 0) continue;  // predecessor not published yet: spin
          excl += w & VAL;
          if ((w >> 62) == 2) break;
          --pt;
        }
        st[tile] = PRE | (excl + (unsigned long long)kept_total);
      }
      s_excl = (int64_t)excl;
    }
    __syncthreads();
  }
  const int64_t out_base = emit ? s_excl : 0;
  int64_t kr = tile_node[tile];
  int64_t rs = e0;
  int64_t kept_run = 0;
  rounds = 0;
  while (rs < e1) {
    ++rounds;
    // a single-round tile keeps its table and staged windows from the count pass
    const bool reuse = emit && single_round;
    int nseg = nseg_saved;
    if (!reuse) {
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
          const T* ta = t + b;
          const T* tb = t + b + la;
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
    nseg = __syncthreads_count(valid);
    // window offsets (exclusive scan of alen + blen over the segments)
    int wlen = (tid < nseg) ? seg[tid].alen + seg[tid].blen : 0;
    int woff, wtot;
    Scan(scan_tmp).ExclusiveSum(wlen, woff, wtot);
    if (tid < nseg) {
      seg[tid].aoff = woff;
      seg[tid].boff = woff + seg[tid].alen;
      seg_pos[tid] = (int)(seg[tid].base + seg[tid].m0 - rs);
    }
    if (tid == 0) {
      const Seg& last = seg[nseg - 1];
      s_round_end = last.base + last.m1;
      s_next_node = kr + nseg;
      seg_pos[nseg] = (int)(s_round_end - rs);
    }
    __syncthreads();
    // ---- 2. stage the input windows (flattened over all segments; coalesced within each
    //        window, every thread busy even when the tile holds many small nodes)
    {
      int sgw = 0;
#pragma unroll 2
      for (int w = tid; w < wtot; w += LTH) {
        while (sgw + 1 < nseg && seg[sgw + 1].aoff <= w) ++sgw;  // w increases per thread
        const int boff = seg[sgw].boff;
        const int64_t gi = (w < boff) ? seg[sgw].ga + (w - seg[sgw].aoff) : seg[sgw].gb + (w - boff);
        s_t[w] = t[gi];
        s_v[w] = v[gi];
        if (MOM) s_v2[w] = v2[gi];
      }
    }
    __syncthreads();
    nseg_saved = nseg;
    }  // !reuse
    const int64_t re = s_round_end;
    // ---- 3. walk LPT positions per thread (twice in the write pass: count, then emit)
    const int p0 = tid * LPT;  // round-relative
    const int rlen = (int)(re - rs);
    auto walk = [&](bool emit, int64_t pos) -> int {
      int nk = 0;
      if (p0 >= rlen) return 0;
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
      for (int q = 0; q < LPT; ++q) {
        const int p = p0 + q;
        if (p >= rlen) break;
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
        if (emit && m == 0) off_out[g.node] = pos;  // node start: first candidate, always kept
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
        if (kp) {
          if (emit) {
            t_out[pos] = tt;
            v_out[pos] = val;
            if (MOM) v2_out[pos] = val2;
            ++pos;
          } else if (!MOM && !isfinite((double)val)) {
            atomicOr(status, 1);
          }
          ++nk;
        }
      }
      return nk;
    };
    int koff, ktot;
    if (emit && single_round) {
      koff = koff_saved;
      ktot = (int)kept_total;
    } else {
      const int nkeep = walk(false, 0);
      Scan(scan_tmp).ExclusiveSum(nkeep, koff, ktot);
      koff_saved = koff;
    }
    if (emit) walk(true, out_base + kept_run + koff);
    kept_run += ktot;
    rs = re;
    kr = s_next_node;
    __syncthreads();  // shared tables are rebuilt next round
  }
  if (!emit) {
    kept_total = kept_run;
    single_round = (rounds == 1);
  }
  }
  if (tid == 0 && e1 == ntot) off_out[nout] = s_excl + kept_total;
}

// Merge-path partition: for every tile start (and the end of the last tile) the output
// node containing it (largest k with off[src[k]] <= e) and the co-rank (A elements among
// the node's first m candidates).
template <typename T>
__global__ void k_tile_part(const T* __restrict__ t, const int64_t* __restrict__ off,
                            const int64_t* __restrict__ src, const int32_t* __restrict__ cnt,
                            int64_t nout, int64_t ntot, int64_t ntiles,
                            int64_t* __restrict__ tile_node, int64_t* __restrict__ tile_i) {
  ntot = off[src[nout - 1] + cnt[nout - 1]];  // live point count (ntot: upper bound)
  for (int64_t tl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; tl <= ntiles;
       tl += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = min(tl * (int64_t)LT, ntot);
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
  const int64_t ntiles = (ntot + LT - 1) / LT;
  size_t cub_b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_b, (const int64_t*)nullptr, (int64_t*)nullptr,
                                (int64_t)(ntiles > 0 ? ntiles : 1));
  *bytes = (int64_t)(4 * 8 * (ntiles + 1) + cub_b + 256 + 16);
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
    cudaMemsetAsync(off_out_dev, 0, (nout + 1) * sizeof(int64_t), s);
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
  cudaMemsetAsync(tile_status, 0, (ntiles + 1) * 8 + 16, s);
  const int pg = (int)((ntiles + 1 + 255) / 256);
  const unsigned grid = (unsigned)ntiles;
#define PCF_TL(T, K, W)                                                                       \
  do {                                                                                        \
    typedef typename std::conditional<K == K_MOM, double, T>::type VT_;                      \
    const int dsm = WCAP * (int)(sizeof(VT_) + sizeof(T) + (K == K_MOM ? sizeof(double) : 0)); \
    cudaFuncSetAttribute(k_level_tiled<T, K, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         dsm);                                                                \
    k_level_tiled<T, K, W><<<grid, LTH, dsm, s>>>(                                            \
        (const T*)t_dev, v_dev, v2_dev, off_dev, src_dev, cnt_dev, leaves_dev, nout, ntot,   \
        tile_node, tile_i, tile_counter, tile_status, (T*)t_out_dev, v_out_dev, v2_out_dev,   \
        off_out_dev, status_dev);                                                             \
  } while (0)
#define PCF_TL_BOTH(T, K)                                                                     \
  do {                                                                                        \
    k_tile_part<T><<<pg, 256, 0, s>>>((const T*)t_dev, off_dev, src_dev, cnt_dev, nout, ntot, \
                                      ntiles, tile_node, tile_i);                             \
    PCF_TL(T, K, true);                                                                       \
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

}  // extern "C"
