// Fused non-compacting tree levels (K5w): k reduction-tree levels in ONE pass over HBM.
//
// Above level 0 of a tree whose breakpoints are (nearly) distinct, every level is a pure
// merge (k_merge_level, pcf_level.cu): each output node is the time-ordered union of its
// two children, every point carrying op(value of A, value of B) at that point, A first on
// ties (reduce.py:31-63 per cell; reduce.py:189-208 for the tree).  One level costs a
// full read + write of every point (3.2 GB at c5), and 19 levels dominate mean / std.
//
// Here one pass runs k levels: an output node at level L+k has C <= 2^k input nodes at
// level L (a contiguous node range, combined in the reference tree shape: pairs
// (0,1)(2,3)..., an odd last node passing through -- the global pairing restricted to
// the subtree).  Its points, in merged order, are the union of the children's points
// ordered by the key (t, child, index) -- exactly what k successive stable merges
// produce.  The node is cut into tiles by keys (pivots taken from its largest child);
// a tile = per child a sub-range [lo_c, hi_c) of points.  Each CTA stages its tile's
// child ranges in shared memory and runs the k pairwise merges there (ping-pong
// buffers), then writes the merged tile once.
//
// Values across a tile boundary: the value of list X just before the tile ("carry") is
// v[lo - 1] for an input child (v[0] when lo = 0: reduce_pair's t = 0 convention, see
// k_merge_level), and combine(carry_A, carry_B) for a merged list -- which is also the
// value of X's first point when nothing of X precedes the tile.  Inside the tile an A
// point takes B's value from B's previous point in the tile or B's carry, and vice
// versa, so every point gets the value the level-by-level path computes, bit for bit
// (same operand order, same rounding to the record kind after every level).
//
// A tile whose child ranges exceed the shared-memory capacity (pivots from one child do
// not bound the other children's counts) is cut further inside the CTA by keys from its
// largest contributor (halving it each time) and processed as consecutive sub-windows,
// so any input -- including long runs of equal times -- is handled.
#include <string.h>
#include <type_traits>
#include "pcf_common.cuh"
#include "pcf_internal.h"

namespace pcfb {
namespace wm {

constexpr int WTH = 256;   // threads per tile CTA (192, or 128 with 1024-point tiles, and 2048-point tiles at 2 CTAs/SM all measured slower)
#ifndef PCF_WLPT_MOM
#define PCF_WLPT_MOM 8
#endif
#ifndef PCF_WLPT
#define PCF_WLPT 8
#endif
#ifndef PCF_WM_PRED
#define PCF_WM_PRED 1
#endif
#ifndef PCF_WM_MOM16
#define PCF_WM_MOM16 1
#endif
constexpr int KMAXC = 16;  // children per output node (k <= 4 levels per pass)
constexpr int kTreeTgt = 512;  // points per K5t tile (one thread each)
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

// points per tile (target) and shared-memory capacity per buffer
template <typename T, int K> struct Cfg {
  static constexpr bool MOM = K == K_MOM;
  static constexpr int CAP = MOM ? 1280 : 2048;  // 3 CTAs per SM (~70 KB each)
  static constexpr int TGT = MOM ? 1024 : 1536;
  using VT = typename std::conditional<MOM, double, T>::type;
  static constexpr int EB = (int)(sizeof(T) + sizeof(VT) + (MOM ? 8 : 0));
  static constexpr int CAPP = CAP + CAP / 8;  // padded slots (pad(x) = x + x / 8)
  static constexpr int SMEM = 2 * CAPP * EB;
  static constexpr int LPT = MOM ? PCF_WLPT_MOM : PCF_WLPT;  // merge positions per thread per round
};

// number of child c's points with key < (T, cs, is): the key order is (t, child, index)
template <typename T>
__device__ __forceinline__ int key_lower(const T* __restrict__ tc, int c, double kt, int cs,
                                         int ki, int lo, int hi) {
  if (c == cs) return ki;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const double x = (double)tc[mid];
    const bool before = c < cs ? (x <= kt) : (x < kt);
    if (before) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// per output node: tile count (>= 1) from its point count
__global__ void k_wnodes(const int64_t* __restrict__ off, const int64_t* __restrict__ nfirst,
                         const int32_t* __restrict__ ncnt, int64_t nout, int64_t tgt,
                         int64_t* __restrict__ tcount, int64_t* __restrict__ off_out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q <= nout;
       q += (int64_t)gridDim.x * blockDim.x) {
    if (q == nout) {
      off_out[nout] = off[nfirst[nout - 1] + ncnt[nout - 1]];
      continue;
    }
    const int64_t f = nfirst[q];
    const int64_t n = off[f + ncnt[q]] - off[f];
    off_out[q] = off[f];
    tcount[q] = n > 0 ? (n + tgt - 1) / tgt : 1;
  }
}

// per-tile descriptors, so a tile CTA needs one dependent load before its staging loads:
// the node's first input node and child count, and per child its input start and the
// tile's [lo, end) range
struct TileHead {
  int64_t f;  // first input node
  int32_t C;
  int32_t pad_;
};
struct TileChild {
  int64_t cb;  // input position of the child's first point
  int32_t lo, end;
};

__global__ void k_wtiles(const int64_t* __restrict__ off, const int64_t* __restrict__ nfirst,
                         const int32_t* __restrict__ ncnt, const int64_t* __restrict__ tbase,
                         const int32_t* __restrict__ rb, int64_t nout,
                         TileHead* __restrict__ th, TileChild* __restrict__ tc) {
  const int64_t ntl = tbase[nout];
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < ntl * KMAXC;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tl = x / KMAXC;
    const int c = (int)(x % KMAXC);
    int64_t lo = 0, hi = nout - 1;  // node: largest q with tbase[q] <= tl
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (tbase[mid] <= tl) lo = mid;
      else hi = mid - 1;
    }
    const int64_t q = lo, f = nfirst[q];
    const int C = ncnt[q];
    if (c == 0) {
      TileHead h;
      h.f = f;
      h.C = C;
      h.pad_ = 0;
      th[tl] = h;
    }
    if (c < C) {
      const int64_t g0 = tl + q;
      TileChild e;
      e.cb = off[f + c];
      e.lo = rb[g0 * KMAXC + c];
      e.end = rb[(g0 + 1) * KMAXC + c];
      tc[tl * KMAXC + c] = e;
    }
  }
}

// single-CTA exclusive scan of n int64 counts -> out[0..n] (n up to a few million)
__global__ void __launch_bounds__(1024) k_scan1(const int64_t* __restrict__ in, int64_t n,
                                                int64_t* __restrict__ out) {
  __shared__ int64_t wsum[32];
  const int tid = threadIdx.x;
  const int64_t per = (n + 1023) / 1024;
  const int64_t b = min((int64_t)tid * per, n), e = min(b + per, n);
  int64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += in[i];
  // block exclusive scan of s
  int64_t x = s;
  const int lane = tid & 31, w = tid >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t z = wsum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    wsum[lane] = z;
  }
  __syncthreads();
  int64_t run = x - s + (w > 0 ? wsum[w - 1] : 0);
  for (int64_t i = b; i < e; ++i) {
    out[i] = run;
    run += in[i];
  }
  if (tid == 1023) out[n] = run;
}

// per (output node, child): the length of the child's leading run of the node's first time
// t0 (every PCF starts at t = 0, so at level L a node begins with one t = 0 point per
// level-0 node -- a tie run that pivots from a single child cannot split)
template <typename T>
__global__ void k_wruns(const T* __restrict__ t, const int64_t* __restrict__ off,
                        const int64_t* __restrict__ nfirst, const int32_t* __restrict__ ncnt,
                        int64_t nout, int32_t* __restrict__ rr) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < nout * KMAXC;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = x / KMAXC;
    const int c = (int)(x % KMAXC);
    const int C = ncnt[q];
    if (c >= C) continue;
    const int64_t f = nfirst[q];
    double t0 = INFINITY;
    for (int d = 0; d < C; ++d)
      if (off[f + d + 1] > off[f + d]) t0 = fmin(t0, (double)t[off[f + d]]);
    const T* tc = t + off[f + c];
    const int nc = (int)(off[f + c + 1] - off[f + c]);
    int lo = 0, hi = nc;  // count of points with t <= t0 (exponential then binary search)
    int step = 1;
    while (step < nc && (double)tc[step] <= t0) step <<= 1;
    lo = step >> 1;
    hi = min(step, nc);
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((double)tc[mid] <= t0) lo = mid + 1;
      else hi = mid;
    }
    rr[q * KMAXC + c] = nc > 0 && (double)tc[0] <= t0 ? lo : 0;
  }
}

// tile boundaries: node q's boundary j (0 .. tcount[q]) lives at global index
// tbase[q] + q + j; per child the number of its points before the boundary key
//
// Boundary j targets merged position P = j * N / ntiles.  Inside the leading t0 run the
// merged order is child by child, so P maps to an exact key (t0, c, P - run prefix);
// past it, the pivot is the largest child's point at the proportional index of the rest.
template <typename T, int K>
__global__ void k_wbounds(const T* __restrict__ t, const int64_t* __restrict__ off,
                          const int64_t* __restrict__ nfirst, const int32_t* __restrict__ ncnt,
                          int64_t nout, const int64_t* __restrict__ tbase,
                          const int32_t* __restrict__ rr, int32_t* __restrict__ rb) {
  const int64_t nb = tbase[nout] + nout;  // boundaries in total
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < nb * KMAXC;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = x / KMAXC;
    const int c = (int)(x % KMAXC);
    int64_t lo = 0, hi = nout - 1;  // node: largest q with tbase[q] + q <= g
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (tbase[mid] + mid <= g) lo = mid;
      else hi = mid - 1;
    }
    const int64_t q = lo;
    const int C = ncnt[q];
    if (c >= C) continue;
    const int64_t j = g - (tbase[q] + q);
    const int64_t nt = tbase[q + 1] - tbase[q];
    const int64_t f = nfirst[q];
    const int nc = (int)(off[f + c + 1] - off[f + c]);
    int r;
    if (j == 0) {
      r = 0;
    } else if (j >= nt) {
      r = nc;
    } else {
      const int64_t N = off[f + C] - off[f];
      const int64_t P = j * N / nt;
      int64_t R = 0;
      for (int d = 0; d < C; ++d) R += rr[q * KMAXC + d];
      int cb = 0, ki;
      double kt;
      if (P < R) {  // inside the leading run: exact
        int64_t pre = 0;
        while (pre + rr[q * KMAXC + cb] <= P) pre += rr[q * KMAXC + cb++];
        ki = (int)(P - pre);
        kt = (double)t[off[f + cb] + ki];
      } else {
        int64_t nbig = -1;
        for (int d = 0; d < C; ++d) {
          const int64_t n = off[f + d + 1] - off[f + d] - rr[q * KMAXC + d];
          if (n > nbig) { nbig = n; cb = d; }
        }
        const int64_t r0 = rr[q * KMAXC + cb];
        ki = (int)(r0 + (P - R) * nbig / (N - R));
        kt = (double)t[off[f + cb] + ki];
      }
      r = key_lower<T>(t + off[f + c], c, kt, cb, ki, 0, nc);
    }
    rb[g * KMAXC + c] = r;
  }
}

__device__ __forceinline__ int pad(int x) { return x + (x >> 3); }  // WLPT = 8

template <typename T, int K>
__global__ void __launch_bounds__(WTH, 3)
    k_wmerge(const T* __restrict__ t, const void* __restrict__ v_, const double* __restrict__ v2,
             const int64_t* __restrict__ off, const int64_t* __restrict__ nfirst,
             const int32_t* __restrict__ ncnt, const int64_t* __restrict__ leaves, int64_t nout,
             int nlev, const int64_t* __restrict__ tbase, const TileHead* __restrict__ th,
             const TileChild* __restrict__ tc,
             T* __restrict__ t_out, void* __restrict__ v_out_, double* __restrict__ v2_out) {
  using C_ = Cfg<T, K>;
  using VT = typename C_::VT;
  constexpr bool MOM = C_::MOM;
  constexpr int CAP = C_::CAP;
  const VT* __restrict__ v = reinterpret_cast<const VT*>(v_);
  VT* __restrict__ v_out = reinterpret_cast<VT*>(v_out_);
  extern __shared__ __align__(16) unsigned char dyn[];
  // buffer k: t[CAP] | v[CAP] | (v2[CAP])
  constexpr int CP = C_::CAPP;
  auto bt = [&](int k) { return reinterpret_cast<T*>(dyn + k * CP * C_::EB); };
  auto bv = [&](int k) {
    return reinterpret_cast<VT*>(dyn + k * CP * C_::EB + CP * (int)sizeof(T));
  };
  auto b2 = [&](int k) {
    return reinterpret_cast<double*>(dyn + k * CP * C_::EB + CP * (int)(sizeof(T) + sizeof(VT)));
  };
  // moments tree, paired layout: (mean, M2) of a point side by side as one 16-byte slot
  // in the value region (same bytes as v[CP] | v2[CP]): one 16-byte load and store per
  // merge step instead of two 8-byte ones each
  constexpr bool P2 = MOM && PCF_WM_MOM16;
  auto bp = [&](int k) {
    return reinterpret_cast<double2*>(dyn + k * CP * C_::EB + CP * (int)sizeof(T));
  };
  __shared__ int64_t s_cb[KMAXC];                 // first input position of each child
  __shared__ int s_lo[KMAXC], s_hi[KMAXC], s_end[KMAXC];
  __shared__ int s_ls[2][KMAXC + 1];              // s_ls[0]: children spans in the buffers
  __shared__ VT s_cv[5][KMAXC];                   // carries per level and list (0: children)
  __shared__ double s_c2[5][KMAXC];
  __shared__ double s_lv[5][KMAXC];               // leaf counts (moments weights)
  __shared__ int s_tot, s_big, s_ki;
  __shared__ double s_kt;
  __shared__ int64_t s_wbase;

  __shared__ int64_t s_f;
  __shared__ int s_C;
  const int tid = threadIdx.x;
  const int64_t ntiles = tbase[nout];
  // persistent: tiles blockIdx.x, blockIdx.x + gridDim.x, ...; the next tile's descriptor
  // is loaded while the current one is processed
  int64_t tl = blockIdx.x;
  if (tl >= ntiles) return;
  TileHead nh = th[tl];
  TileChild nc_;
  if (tid < KMAXC && tid < nh.C) nc_ = tc[tl * KMAXC + tid];
  for (; tl < ntiles; tl += gridDim.x) {
  if (tid == 0) {
    s_f = nh.f;
    s_C = nh.C;
  }
  if (tid < nh.C) {
    s_cb[tid] = nc_.cb;
    s_lo[tid] = nc_.lo;
    s_end[tid] = nc_.end;
  }
  __syncthreads();
  const int64_t f = s_f;
  const int C = s_C;
  const int64_t nbase = s_cb[0];
  if (tl + gridDim.x < ntiles) {  // prefetch the next descriptor
    nh = th[tl + gridDim.x];
    if (tid < KMAXC && tid < nh.C) nc_ = tc[(tl + gridDim.x) * KMAXC + tid];
  }
  if (MOM && tid < C) s_lv[0][tid] = (double)leaves[f + tid];
  __syncthreads();
  for (;;) {
    // ---- the next sub-window [lo, hi): the whole tile unless it exceeds CAP points
    if (tid < C) s_hi[tid] = s_end[tid];
    __syncthreads();
    for (;;) {
      if (tid == 0) {
        int tot = 0, big = 0, nbig = -1;
        for (int c = 0; c < C; ++c) {
          const int n = s_hi[c] - s_lo[c];
          tot += n;
          if (n > nbig) { nbig = n; big = c; }
        }
        s_tot = tot;
        if (tot > CAP) {
          const int mid = s_lo[big] + nbig / 2;
          s_big = big;
          s_ki = mid;
          s_kt = (double)t[s_cb[big] + mid];
        }
      }
      __syncthreads();
      if (s_tot <= CAP) break;
      if (tid < C)
        s_hi[tid] = key_lower<T>(t + s_cb[tid], tid, s_kt, s_big, s_ki, s_lo[tid], s_hi[tid]);
      __syncthreads();
    }
    const int E = s_tot;
    if (tid == 0) {
      int run = 0;
      int64_t wb = 0;
      for (int c = 0; c < C; ++c) {
        s_ls[0][c] = run;
        run += s_hi[c] - s_lo[c];
        wb += s_lo[c];
      }
      s_ls[0][C] = run;
      s_wbase = wb;
    }
    __syncthreads();
    // ---- the k levels, warp groups per list: at level L (1..D, D = ceil(log2 C)) output
    //      list i holds children [i 2^L, (i+1) 2^L) and is merged by warps
    //      [i g, (i+1) g), g = 8 >> (D - L); those warps produced its two inputs at level
    //      L - 1 (or staged its children), so they sync among themselves only (named
    //      barriers) -- one CTA barrier per tile instead of one per level
    const int D = C > 1 ? 32 - __clz(C - 1) : 0;  // levels that combine anything
    const int warp = tid >> 5;
    auto group_sync = [&](int gsz, int grp) {
      if (gsz == 1) {
        __syncwarp();
      } else if (gsz == WTH / 32) {
        __syncthreads();
      } else {  // ids 1..4 for pairs of warps, 5..6 for quads
        const int id = (gsz == 2 ? 1 : 5) + grp;
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(gsz * 32) : "memory");
      }
    };
    {
      // staging: the level-1 group of list j stages children 2j, 2j + 1 (and their carries)
      const int g1 = D > 0 ? (WTH / 32) >> (D - 1) : WTH / 32;
      const int grp = warp / g1, r = tid - grp * g1 * 32;
      T* st = bt(0);
      VT* sv = bv(0);
      double* s2 = b2(0);
      const int c0 = D > 0 ? 2 * grp : 0, c1 = D > 0 ? min(2 * grp + 2, C) : C;
      for (int c = c0; c < c1; ++c) {
        const int x0 = s_ls[0][c], x1 = s_ls[0][c + 1];
        const T* gt = t + (s_cb[c] + s_lo[c] - x0);
        const VT* gv = v + (s_cb[c] + s_lo[c] - x0);
        const double* g2 = v2 + (s_cb[c] + s_lo[c] - x0);
        for (int x = x0 + r; x < x1; x += g1 * 32) {
          const int y = pad(x);
          cp_async_rec<sizeof(T)>(smem_u32(st + y), gt + x);
          if (P2) {
            const uint32_t pa = smem_u32(bp(0) + y);
            cp_async_rec<8>(pa, gv + x);
            cp_async_rec<8>(pa + 8u, g2 + x);
          } else {
            cp_async_rec<sizeof(VT)>(smem_u32(sv + y), gv + x);
            if (MOM) cp_async_rec<8>(smem_u32(s2 + y), g2 + x);
          }
        }
        if (r == 0) {  // the child's point before the window (its first point at 0)
          const int64_t pc = s_cb[c] + (s_lo[c] > 0 ? s_lo[c] - 1 : 0);
          cp_async_rec<sizeof(VT)>(smem_u32(&s_cv[0][c]), v + pc);
          if (MOM) {
            cp_async_rec<8>(smem_u32(&s_c2[0][c]), v2 + pc);
            s_lv[0][c] = (double)leaves[f + c];
          }
        }
      }
      cp_async_commit();
      cp_async_wait<0>();
      if (D > 0) group_sync(g1, grp);
    }
    const T TINF = (T)INFINITY;
    for (int L = 1; L <= D; ++L) {
      const int gsz = (WTH / 32) >> (D - L);
      const int li = warp / gsz;                 // this group's output list
      const int ca0 = li << L;                   // its first child
      if (L > 1) group_sync(gsz, li);            // its inputs (level L - 1) are complete
      if (ca0 >= C) continue;                    // an empty list: nothing to merge
      const int cmid = min(ca0 + (1 << (L - 1)), C), cend = min(ca0 + (1 << L), C);
      const bool pass = cmid >= C;               // right subtree empty: passthrough
      const int a0 = s_ls[0][ca0], b0 = s_ls[0][cmid], e0 = s_ls[0][cend];
      const int na = b0 - a0, nb = e0 - b0;
      // carries (and leaf counts) of the inputs: lists 2 li and 2 li + 1 of level L - 1
      const VT cva = s_cv[L - 1][2 * li];
      const VT cvb = pass ? VT(0) : s_cv[L - 1][2 * li + 1];
      const double c2a = MOM ? s_c2[L - 1][2 * li] : 0.0;
      const double c2b = (MOM && !pass) ? s_c2[L - 1][2 * li + 1] : 0.0;
      double wB = 0.0, wAB = 0.0;
      if (MOM && !pass) {
        const double nA = s_lv[L - 1][2 * li], nB = s_lv[L - 1][2 * li + 1];
        const double n = nA + nB;
        wB = nB / n;
        wAB = nA * nB / n;
      }
      const int r = tid - li * gsz * 32;         // rank in the group
      if (r == 0) {  // this list's carry and leaf count for level L + 1
        if (pass) {
          s_cv[L][li] = cva;
          if (MOM) {
            s_c2[L][li] = c2a;
            s_lv[L][li] = s_lv[L - 1][2 * li];
          }
        } else if (MOM) {
          const double d = (double)cvb - (double)cva;
          s_cv[L][li] = (VT)((double)cva + d * wB);
          s_c2[L][li] = (c2a + c2b) + d * d * wAB;
          s_lv[L][li] = s_lv[L - 1][2 * li] + s_lv[L - 1][2 * li + 1];
        } else {
          s_cv[L][li] = to_t<VT>(vop<K>((double)cva, (double)cvb));
        }
      }
      const T* it = bt((L - 1) & 1);
      const VT* iv = bv((L - 1) & 1);
      const double* i2 = b2((L - 1) & 1);
      T* ot = bt(L & 1);
      VT* ov = bv(L & 1);
      double* o2 = b2(L & 1);
      constexpr int WLPT = C_::LPT;
      if (pass) {  // right subtree empty: the list is copied (its values are its own)
        for (int x = r; x < na; x += gsz * 32) {
          const int y = pad(a0 + x);
          ot[y] = it[y];
          if (P2) {
            bp(L & 1)[y] = bp((L - 1) & 1)[y];
          } else {
            ov[y] = iv[y];
            if (MOM) o2[y] = i2[y];
          }
        }
        continue;
      }
      for (int base = 0; base < na + nb; base += gsz * 32 * WLPT) {
        const int m0 = base + r * WLPT;          // first output position (list-relative)
        if (m0 >= na + nb) break;
        int lo = max(0, m0 - nb), hi = min(m0, na);
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (it[pad(a0 + mid)] <= it[pad(b0 + m0 - mid - 1)]) lo = mid + 1;
          else hi = mid;
        }
        int i = lo;  // A points consumed; B points consumed = (output position) - i
        T tai = i < na ? it[pad(a0 + i)] : TINF;
        T tbj = m0 - i < nb ? it[pad(b0 + m0 - i)] : TINF;
        VT ca, cb;
        double ca2, cb2;
        const double2* ip = bp((L - 1) & 1);
        double2* op = bp(L & 1);
        if (P2) {
          const double2 pa = i > 0 ? ip[pad(a0 + i - 1)] : make_double2((double)cva, c2a);
          const double2 pb = m0 - i > 0 ? ip[pad(b0 + m0 - i - 1)] : make_double2((double)cvb, c2b);
          ca = (VT)pa.x; ca2 = pa.y;
          cb = (VT)pb.x; cb2 = pb.y;
        } else {
          ca = i > 0 ? iv[pad(a0 + i - 1)] : cva;
          cb = m0 - i > 0 ? iv[pad(b0 + m0 - i - 1)] : cvb;
          ca2 = MOM ? (i > 0 ? i2[pad(a0 + i - 1)] : c2a) : 0.0;
          cb2 = MOM ? (m0 - i > 0 ? i2[pad(b0 + m0 - i - 1)] : c2b) : 0.0;
        }
        // one merge step at output position m = m0 + q, branch-free: the consumed list's
        // point (value) and its next time are the only loads; selects route them to A's
        // or B's state.  The output buffer is the other ping-pong half.
        auto step = [&](int m, bool live) {
          const bool takeA = tai <= tbj;  // A first on ties
          const int x = takeA ? a0 + i : b0 + (m - i);
          const int xe = takeA ? b0 : e0;
          const int y = pad(a0 + m);
          if (live) ot[y] = takeA ? tai : tbj;
          double2 pv;
          if (P2) pv = ip[pad(x)];
          const VT val = P2 ? (VT)pv.x : iv[pad(x)];
          const T nt = x + 1 < xe ? it[pad(x + 1)] : TINF;
          ca = takeA ? val : ca;
          cb = takeA ? cb : val;
          tai = takeA ? nt : tai;
          tbj = takeA ? tbj : nt;
          // past the list's end both times are +inf and takeA holds: i stops at na, so
          // the dead steps re-read B's first point (this list's own input, never another
          // group's) and store nothing
          i += (takeA && i < na) ? 1 : 0;
          if (MOM) {
            const double v2x = P2 ? pv.y : i2[pad(x)];
            ca2 = takeA ? v2x : ca2;
            cb2 = takeA ? cb2 : v2x;
            const double d = (double)cb - (double)ca;
            if (live) {
              if (P2) {
                op[y] = make_double2((double)ca + d * wB, (ca2 + cb2) + d * d * wAB);
              } else {
                ov[y] = (VT)((double)ca + d * wB);
                o2[y] = (ca2 + cb2) + d * d * wAB;
              }
            }
          } else {
            if (live) ov[y] = to_t<VT>(vop<K>((double)ca, (double)cb));
          }
        };
#if PCF_WM_PRED
        // one unrolled body, the list's tail handled by predicated stores (no per-step
        // branch and reconvergence)
#pragma unroll
        for (int q = 0; q < WLPT; ++q) step(m0 + q, m0 + q < na + nb);
#else
        // (one guarded unrolled loop: splitting off an unguarded full-WLPT path measured
        // slower, 14.6 vs 13.9 ms on c5 mean)
#pragma unroll
        for (int q = 0; q < WLPT; ++q)
          if (m0 + q < na + nb) step(m0 + q, true);
#endif
      }
    }
    __syncthreads();
    const int cur = D & 1;
    // ---- the merged window, written once (coalesced)
    {
      const T* st = bt(cur);
      const VT* sv = bv(cur);
      const double* s2 = b2(cur);
      const int64_t ob = nbase + s_wbase;
      for (int x = tid; x < E; x += WTH) {
        const int y = pad(x);
        t_out[ob + x] = st[y];
        if (P2) {
          const double2 w = bp(cur)[y];
          v_out[ob + x] = (VT)w.x;
          v2_out[ob + x] = w.y;
        } else {
          v_out[ob + x] = sv[y];
          if (MOM) v2_out[ob + x] = s2[y];
        }
      }
    }
    // ---- next sub-window of the tile
    __syncthreads();
    int more = 0;
    if (tid < C) {
      s_lo[tid] = s_hi[tid];
      more = s_lo[tid] < s_end[tid];
    }
    if (!__syncthreads_or(more)) break;
    if (MOM && tid < C) s_lv[0][tid] = (double)leaves[f + tid];
  }
  __syncthreads();  // the descriptors in shared memory are reused by the next tile
  }
}

// ---------------------------------------------------------------------------------------
// K5t: the same fused levels as a streaming merge tree per THREAD.  One thread owns one
// tile (the key-ordered window of an output node, same tiles as K5w) and pulls its points
// in order through a static binary tree of 2-way mergers held in registers: a merger keeps
// the next point of each input (time + value) and each input's current value; next() takes
// the input whose next point comes first (A on ties), refills it from below and returns
// (t, combine(cur_A, cur_B)) -- a passthrough merger (empty right subtree) returns cur_A.
// The leaves read their child's points from global memory.  No shared memory, barriers or
// co-rank searches: ~D compares and D combines per output point for D levels.  Measured
// slower than K5w (each thread streams 2^D lists from global memory, uncoalesced; 186
// registers at D = 3), so it is opt-in: PCF_TREE_KERNEL=tree.
template <typename T, int K, int D>
struct MNode {
  MNode<T, K, D - 1> a, b;
  T ta, tb;       // next point times of a and b (+inf when exhausted)
  T va, vb;       // values of those next points
  T ca, cb;       // current values of a and b
  bool hasb;      // right subtree holds at least one child
  __device__ __forceinline__ void init(const T* __restrict__ t, const T* __restrict__ v,
                                       const int64_t* cbase, const int* lo, const int* en,
                                       int C, int first, T* carry) {
    hasb = first + (1 << (D - 1)) < C;
    T cra, crb;
    a.init(t, v, cbase, lo, en, C, first, &cra);
    b.init(t, v, cbase, lo, en, C, first + (1 << (D - 1)), &crb);
    ca = cra;
    cb = crb;
    *carry = hasb ? to_t<T>(vop<K>((double)cra, (double)crb)) : cra;
    a.next(ta, va);
    b.next(tb, vb);
  }
  __device__ __forceinline__ void next(T& t, T& v) {
    if (ta <= tb) {  // A first on ties
      t = ta;
      ca = va;
      a.next(ta, va);
    } else {
      t = tb;
      cb = vb;
      b.next(tb, vb);
    }
    v = hasb ? to_t<T>(vop<K>((double)ca, (double)cb)) : ca;
  }
};

template <typename T, int K>
struct MNode<T, K, 0> {  // one child of the output node: its window [pos, end) in global
  const T* __restrict__ tp;
  const T* __restrict__ vp;
  int pos, end;
  __device__ __forceinline__ void init(const T* __restrict__ t, const T* __restrict__ v,
                                       const int64_t* cbase, const int* lo, const int* en,
                                       int C, int first, T* carry) {
    if (first < C) {
      tp = t + cbase[first];
      vp = v + cbase[first];
      pos = lo[first];
      end = en[first];
      *carry = vp[pos > 0 ? pos - 1 : 0];  // reduce_pair's t = 0 convention at pos 0
    } else {  // no such child
      tp = t;
      vp = v;
      pos = end = 0;
      *carry = (T)0;
    }
  }
  __device__ __forceinline__ void next(T& t, T& v) {
    if (pos < end) {
      t = tp[pos];
      v = vp[pos];
      ++pos;
    } else {
      t = (T)INFINITY;
      v = (T)0;
    }
  }
};

template <typename T, int K, int D>
__global__ void __launch_bounds__(128)
    k_wtree(const T* __restrict__ t, const T* __restrict__ v, int64_t nout,
            const int64_t* __restrict__ tbase, const TileHead* __restrict__ th,
            const TileChild* __restrict__ tc, T* __restrict__ t_out, T* __restrict__ v_out) {
  const int64_t ntiles = tbase[nout];
  for (int64_t tl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; tl < ntiles;
       tl += (int64_t)gridDim.x * blockDim.x) {
    const TileHead h = th[tl];
    const int C = h.C;
    int64_t cbase[1 << D];
    int lo[1 << D], en[1 << D];
    int64_t count = 0, before = 0;
#pragma unroll
    for (int c = 0; c < (1 << D); ++c) {
      if (c < C) {
        const TileChild e = tc[tl * KMAXC + c];
        cbase[c] = e.cb;
        lo[c] = e.lo;
        en[c] = e.end;
        count += e.end - e.lo;
        before += e.lo;
      } else {
        cbase[c] = 0;
        lo[c] = en[c] = 0;
      }
    }
    MNode<T, K, D> root;
    T carry;
    root.init(t, v, cbase, lo, en, C, 0, &carry);
    const int64_t ob = cbase[0] + before;  // node start (first child's start) + points before
    for (int64_t o = 0; o < count; ++o) {
      T tt, vv;
      root.next(tt, vv);
      t_out[ob + o] = tt;
      v_out[ob + o] = vv;
    }
  }
}

template <typename T, int K>
void launch_tree(int nlev, const T* t, const T* v, int64_t nout, const int64_t* tbase,
                 const TileHead* th, const TileChild* tc, T* t_out, T* v_out, int64_t ntile_max,
                 int nsm, cudaStream_t s) {
  if constexpr (K != K_MOM) {
    const unsigned grid = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>((ntile_max + 127) / 128, (int64_t)nsm * 32));
    if (nlev == 1)
      k_wtree<T, K, 1><<<grid, 128, 0, s>>>(t, v, nout, tbase, th, tc, t_out, v_out);
    else if (nlev == 2)
      k_wtree<T, K, 2><<<grid, 128, 0, s>>>(t, v, nout, tbase, th, tc, t_out, v_out);
    else
      k_wtree<T, K, 3><<<grid, 128, 0, s>>>(t, v, nout, tbase, th, tc, t_out, v_out);
  }
}

// Equal-time coincidences between neighbouring nodes (2p, 2p+1) for nsample pairs spread
// over the level: counts[0] += coincidences, counts[1] += points.  Decides before level 0
// whether the tree can run non-compacting (nearly distinct breakpoints) from the start.
template <typename T>
__global__ void k_dup_sample(const T* __restrict__ t, const int64_t* __restrict__ off,
                             int64_t nnodes, int nsample, unsigned long long* __restrict__ counts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nsample || nnodes < 2) return;
  const int64_t pa = 2 * ((int64_t)i * (nnodes / 2) / nsample);
  const T* a = t + off[pa];
  const T* b = t + off[pa + 1];
  const int64_t na = off[pa + 1] - off[pa], nb = off[pa + 2] - off[pa + 1];
  int64_t x = 0, y = 0;
  unsigned long long dup = 0;
  while (x < na && y < nb) {
    const T u = a[x], w = b[y];
    dup += (u == w);
    x += (u <= w);
    y += (w <= u);
  }
  atomicAdd(&counts[0], dup);
  atomicAdd(&counts[1], (unsigned long long)(na + nb));
}

}  // namespace wm
}  // namespace pcfb

using namespace pcfb;
using namespace pcfb::wm;

extern "C" {

// workspace for pcf_tree_merge_levels: tile counts / bases (nout + 1 each) and the
// boundary table ((ntot / 1280 + 2 * nout + 2) x 16 int32)
int pcf_tree_merge_levels_workspace(int64_t ntot, int64_t nout, int64_t* bytes) {
  if (!bytes || ntot < 0 || nout < 0) {
    set_error("pcf_tree_merge_levels_workspace: bad arguments");
    return PCF_ERR_ARG;
  }
  const int64_t nb = ntot / kTreeTgt + 2 * nout + 2;
  const int64_t nt = ntot / kTreeTgt + nout + 1;  // tiles (upper bound)
  *bytes = 2 * (nout + 1) * 8 + nb * KMAXC * 4 + nout * KMAXC * 4 + nt * 16 +
           nt * KMAXC * 16 + 512;
  return PCF_OK;
}

int pcf_tree_merge_levels(int kind, int is_f32, const void* t_dev, const void* v_dev,
                          const double* v2_dev, const int64_t* off_dev,
                          const int64_t* nfirst_dev, const int32_t* ncnt_dev,
                          const int64_t* leaves_dev, int64_t nout, int32_t nlev, int64_t ntot,
                          void* t_out_dev, void* v_out_dev, double* v2_out_dev,
                          int64_t* off_out_dev, void* ws_dev, int64_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (nout <= 0) return PCF_OK;
  if (kind < 0 || kind > 4 || nlev < 1 || nlev > 4 || !t_dev || !v_dev || !off_dev ||
      !nfirst_dev || !ncnt_dev || !t_out_dev || !v_out_dev || !off_out_dev || !ws_dev ||
      (kind == K_MOM && (!v2_dev || !v2_out_dev || !leaves_dev))) {
    set_error("pcf_tree_merge_levels: bad arguments");
    return PCF_ERR_ARG;
  }
  int64_t need = 0;
  pcf_tree_merge_levels_workspace(ntot, nout, &need);
  if (ws_bytes < need) {
    set_error("pcf_tree_merge_levels: workspace %lld < %lld bytes", (long long)ws_bytes,
              (long long)need);
    return PCF_ERR_ARG;
  }
  int64_t* tcount = (int64_t*)ws_dev;
  int64_t* tbase = tcount + (nout + 1);
  int32_t* rr = (int32_t*)(tbase + (nout + 1));
  int32_t* rb = rr + nout * KMAXC;
  const int64_t ntile_max = ntot / kTreeTgt + nout + 1;
  uintptr_t pth = (uintptr_t)(rb + (ntot / kTreeTgt + 2 * nout + 2) * KMAXC);
  pth = (pth + 15) & ~(uintptr_t)15;
  TileHead* th = (TileHead*)pth;
  TileChild* tch = (TileChild*)(th + ntile_max);
  const int ng = (int)std::min<int64_t>((nout + 1 + 255) / 256, 4096);
  const int bg = (int)std::min<int64_t>(((ntile_max + nout + 1) * KMAXC + 255) / 256, 148 * 64);
  const int rg = (int)std::min<int64_t>((nout * KMAXC + 255) / 256, 148 * 64);
  int nsm = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // K5t is opt-in (PCF_TREE_KERNEL=tree): bit-identical, but each thread's eight
  // uncoalesced input streams make it 2.4-3.2x slower than K5w on c5 (40-54 vs 16.7 ms)
  static const bool tree_env = getenv("PCF_TREE_KERNEL") != nullptr &&
                               strcmp(getenv("PCF_TREE_KERNEL"), "tree") == 0;
  const bool tree = tree_env && kind != K_MOM && nlev <= 3;  // K5t (per-thread merge tree)
#define PCF_WM(T, K)                                                                          \
  do {                                                                                        \
    k_wnodes<<<ng, 256, 0, s>>>(off_dev, nfirst_dev, ncnt_dev, nout,                          \
                                tree ? (int64_t)kTreeTgt : (int64_t)Cfg<T, K>::TGT, tcount,    \
                                off_out_dev);                                                 \
    k_scan1<<<1, 1024, 0, s>>>(tcount, nout, tbase);                                          \
    k_wruns<T><<<rg, 256, 0, s>>>((const T*)t_dev, off_dev, nfirst_dev, ncnt_dev, nout, rr);  \
    k_wbounds<T, K><<<bg, 256, 0, s>>>((const T*)t_dev, off_dev, nfirst_dev, ncnt_dev, nout,  \
                                       tbase, rr, rb);                                        \
    k_wtiles<<<bg, 256, 0, s>>>(off_dev, nfirst_dev, ncnt_dev, tbase, rb, nout, th, tch);     \
    if (tree && K != K_MOM) {                                                                 \
      launch_tree<T, K>(nlev, (const T*)t_dev, (const T*)v_dev, nout, tbase, th, tch,          \
                        (T*)t_out_dev, (T*)v_out_dev, ntile_max, nsm, s);                     \
    } else {                                                                                  \
      const int dsm = Cfg<T, K>::SMEM;                                                        \
      cudaFuncSetAttribute(k_wmerge<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, dsm); \
      int per_sm = 0;                                                                         \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_wmerge<T, K>, WTH, dsm);        \
      const int64_t grid =                                                                    \
          std::min<int64_t>(ntot / Cfg<T, K>::TGT + nout + 1, (int64_t)std::max(1, per_sm) * nsm); \
      k_wmerge<T, K><<<(unsigned)grid, WTH, dsm, s>>>(                                        \
          (const T*)t_dev, v_dev, v2_dev, off_dev, nfirst_dev, ncnt_dev, leaves_dev, nout,    \
          nlev, tbase, th, tch, (T*)t_out_dev, v_out_dev, v2_out_dev);                        \
    }                                                                                         \
  } while (0)
  if (is_f32) {
    switch (kind) {
      case K_ADD: PCF_WM(float, K_ADD); break;
      case K_MAX: PCF_WM(float, K_MAX); break;
      case K_MIN: PCF_WM(float, K_MIN); break;
      case K_MUL: PCF_WM(float, K_MUL); break;
      default: PCF_WM(float, K_MOM); break;
    }
  } else {
    switch (kind) {
      case K_ADD: PCF_WM(double, K_ADD); break;
      case K_MAX: PCF_WM(double, K_MAX); break;
      case K_MIN: PCF_WM(double, K_MIN); break;
      case K_MUL: PCF_WM(double, K_MUL); break;
      default: PCF_WM(double, K_MOM); break;
    }
  }
#undef PCF_WM
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("pcf_tree_merge_levels: %s", cudaGetErrorString(e));
    return PCF_ERR_CUDA;
  }
  return PCF_OK;
}

int pcf_tree_dup_sample(int is_f32, const void* t_dev, const int64_t* off_dev, int64_t nnodes,
                        int32_t nsample, unsigned long long* counts_dev, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!t_dev || !off_dev || !counts_dev || nnodes < 0 || nsample < 1) {
    set_error("pcf_tree_dup_sample: bad arguments");
    return PCF_ERR_ARG;
  }
  cudaError_t e = cudaMemsetAsync(counts_dev, 0, 2 * sizeof(unsigned long long), s);
  if (e == cudaSuccess && nnodes >= 2) {
    const int g = (nsample + 127) / 128;
    if (is_f32)
      k_dup_sample<float><<<g, 128, 0, s>>>((const float*)t_dev, off_dev, nnodes, nsample, counts_dev);
    else
      k_dup_sample<double><<<g, 128, 0, s>>>((const double*)t_dev, off_dev, nnodes, nsample,
                                             counts_dev);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    set_error("pcf_tree_dup_sample: %s", cudaGetErrorString(e));
    return PCF_ERR_CUDA;
  }
  return PCF_OK;
}

}  // extern "C"
