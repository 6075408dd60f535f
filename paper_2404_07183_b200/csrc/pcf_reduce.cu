// Reduction path helpers: compaction (scan + scatter) and the mean/std finalisation
// (reduce.py:211-238, core.py:165-214).  The tree levels themselves are in pcf_level.cu.
//
// The finalisation flags every point of the root node(s) -- keep where the scaled value
// differs from the previous surviving point's (minimize_discretization), drop zero-width
// pieces left by non-compacting levels.  pcf_finalize does it in two passes over tiles of
// 4096 points (count the kept points per tile; single-CTA scan of the tile counts;
// recompute and write the kept points through shared memory, coalesced), so neither the
// scaled values nor the flags ever go to HBM.  pcf_compact (flags -> positions -> scatter)
// uses the same tile scan.  No library scan on this path.
#include <type_traits>
#include "pcf_common.cuh"
#include "pcf_internal.h"

namespace pcfb {

template <typename T> __device__ __forceinline__ T to_t(double x);
template <> __device__ __forceinline__ double to_t<double>(double x) { return x; }
template <> __device__ __forceinline__ float to_t<float>(double x) { return __double2float_rn(x); }

// ------------------------------------------------------------ compaction
template <typename T, typename V>
__global__ void k_scatter(const T* __restrict__ st, const V* __restrict__ sv,
                          const V* __restrict__ sv2, const int32_t* __restrict__ flag,
                          const int64_t* __restrict__ pos, int64_t ntot, T* __restrict__ t_out,
                          V* __restrict__ v_out, V* __restrict__ v2_out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ntot;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (flag[e]) {
      const int64_t p = pos[e];
      t_out[p] = st[e];
      v_out[p] = sv[e];
      if (sv2) v2_out[p] = sv2[e];
    }
  }
}

__global__ void k_out_offsets(const int64_t* __restrict__ off_in, const int64_t* __restrict__ src,
                              int64_t nout, const int64_t* __restrict__ pos,
                              const int32_t* __restrict__ flag, int64_t ntot,
                              int64_t* __restrict__ off_out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= nout;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (k < nout) {
      const int64_t b = off_in[src[k]];
      off_out[k] = b < ntot ? pos[b] : (ntot ? pos[ntot - 1] + flag[ntot - 1] : 0);
    } else {
      off_out[k] = ntot ? pos[ntot - 1] + flag[ntot - 1] : 0;
    }
  }
}

// ------------------------------------------------------------ finalisation (K6)
// mean: v * T(scale) in T arithmetic (core.scale, core.py:172), then keep where the value
// changes (minimize_discretization, core.py:189-203).  Per-segment scale factors allow a
// batch of independent means (mean_along).
// Zero-width pieces (non-compacting levels, k_merge_level): point e is dropped when the
// next point of its node has the same time; a surviving point is compared with the last
// survivor before it, i.e. the point just before its run of equal times.
template <typename T>
__device__ __forceinline__ bool zero_width(const T* __restrict__ t, int64_t e, int64_t end) {
  return t && e + 1 < end && t[e + 1] == t[e];
}

template <typename T>
__device__ __forceinline__ int64_t prev_survivor(const T* __restrict__ t, int64_t e,
                                                 int64_t begin) {
  if (!t || e == begin || t[e - 1] != t[e]) return e - 1;
  // node times are non-decreasing: binary search for the start of e's run of equal times
  // (the t = 0 run of a non-compacting tree holds one point per merged level)
  int64_t lo = begin, hi = e;
  const T te = t[e];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (t[mid] < te) lo = mid + 1;
    else hi = mid;
  }
  return lo - 1;
}

// mean: v * T(scale) in T arithmetic (core.scale, core.py:172), then keep where the value
// changes (minimize_discretization, core.py:189-203).  Per-segment scale factors allow a
// batch of independent means (mean_along).  t (optional): drop zero-width pieces first.
template <typename T>
__global__ void k_scale_flag(const T* __restrict__ v, const T* __restrict__ t,
                             const int64_t* __restrict__ off, int64_t nseg,
                             const double* __restrict__ scale, int64_t ntot,
                             T* __restrict__ sv, int32_t* __restrict__ flag,
                             int32_t* __restrict__ status) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ntot;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nseg - 1;
    while (lo < hi) {
      int64_t mid = (lo + hi + 1) >> 1;
      if (off[mid] <= e) lo = mid;
      else hi = mid - 1;
    }
    const T a = to_t<T>(scale[lo]);
    const T x = v[e] * a;
    sv[e] = x;
    if (zero_width(t, e, off[lo + 1])) {
      flag[e] = 0;
      continue;
    }
    if (!isfinite((double)x)) atomicOr(status, 1);
    const int64_t p = prev_survivor(t, e, off[lo]);
    flag[e] = (p < off[lo]) ? 1 : (x != v[p] * a);
  }
}

// std: s = T(sqrt(double(T(M2 * scale)))) (variance scale in float64, then
// core.apply_unary(math.sqrt)), keep where s changes.
template <typename T, bool SQRT>
__global__ void k_std_flag(const double* __restrict__ m2, const T* __restrict__ t,
                           const int64_t* __restrict__ off, int64_t nseg,
                           const double* __restrict__ scale, int64_t ntot,
                           T* __restrict__ sv, int32_t* __restrict__ flag,
                           int32_t* __restrict__ status) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ntot;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nseg - 1;
    while (lo < hi) {
      int64_t mid = (lo + hi + 1) >> 1;
      if (off[mid] <= e) lo = mid;
      else hi = mid - 1;
    }
    const double sc = scale[lo];
    auto sd = [&](int64_t q) {
      const T var = to_t<T>(m2[q] * sc);
      return SQRT ? to_t<T>(sqrt((double)var)) : var;
    };
    const T x = sd(e);
    sv[e] = x;
    if (zero_width(t, e, off[lo + 1])) {
      flag[e] = 0;
      continue;
    }
    if (!isfinite((double)x)) atomicOr(status, 1);
    const int64_t p = prev_survivor(t, e, off[lo]);
    flag[e] = (p < off[lo]) ? 1 : (x != sd(p));
  }
}


// ------------------------------------------------------------ tiled finalisation
constexpr int FT = 256;           // threads per tile
constexpr int FPT = 8;            // consecutive points per thread
constexpr int FTILE = FT * FPT;   // points per tile

// value of point q (kind 0: mean = v * T(scale); 1: variance T(M2 * scale); 2: std)
template <typename T, int KIND>
__device__ __forceinline__ T fin_value(const void* __restrict__ src, int64_t q, double sc) {
  if (KIND == 0) {
    const T* v = reinterpret_cast<const T*>(src);
    return v[q] * to_t<T>(sc);
  }
  const double* m2 = reinterpret_cast<const double*>(src);
  const T var = to_t<T>(m2[q] * sc);
  return KIND == 2 ? to_t<T>(sqrt((double)var)) : var;
}

// point e: value and keep flag (first point of its node, or a value change against the
// last survivor; zero-width pieces dropped).  The warp's 32 consecutive points load their
// own time and source value once; the neighbours' come by shuffles (one extra load at each
// end of the warp), so a point's loads never wait for another's.
template <typename T, int KIND>
__device__ __forceinline__ bool fin_point(const void* __restrict__ src, const T* __restrict__ t,
                                          int64_t e, int64_t ntot, int64_t sbeg, int64_t send,
                                          double sc, T* val, bool* bad) {
  using SV = typename std::conditional<KIND == 0, T, double>::type;
  const SV* sv = reinterpret_cast<const SV*>(src);
  const int lane = threadIdx.x & 31;
  const bool in = e < ntot;
  const T te = in ? t[e] : (T)0;
  const SV xe = in ? sv[e] : (SV)0;
  T tn = __shfl_down_sync(0xffffffffu, te, 1);
  T tp = __shfl_up_sync(0xffffffffu, te, 1);
  SV xp = __shfl_up_sync(0xffffffffu, xe, 1);
  if (lane == 31 && e + 1 < ntot) tn = t[e + 1];
  if (lane == 0 && e > 0) {
    tp = t[e - 1];
    xp = sv[e - 1];
  }
  auto value = [&](SV x) -> T {
    if (KIND == 0) return (T)x * to_t<T>(sc);
    const T var = to_t<T>((double)x * sc);
    return KIND == 2 ? to_t<T>(sqrt((double)var)) : var;
  };
  const T x = value(xe);
  *val = x;
  if (!in) return false;
  if (t && e + 1 < send && tn == te) return false;  // zero-width piece
  if (!isfinite((double)x)) *bad = true;
  if (e == sbeg) return true;  // first point of its node
  if (!t || tp != te) return x != value(xp);  // the previous point is the last survivor
  const int64_t p = prev_survivor(t, e, sbeg);  // inside a run of equal times (rare)
  return p < sbeg || x != value(sv[p]);
}

// node of point e (largest k with off[k] <= e)
__device__ __forceinline__ int64_t seg_of(const int64_t* __restrict__ off, int64_t nseg,
                                          int64_t e) {
  int64_t lo = 0, hi = nseg - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (off[mid] <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// A tile is FPT rows of FT consecutive points; warp w of row k handles 32 consecutive
// points (coalesced loads), its keep flags are one ballot.  Point order = (row, warp, lane).
template <typename T, int KIND>
__global__ void __launch_bounds__(FT, 4) k_fin_count(const void* __restrict__ src,
                                                  const T* __restrict__ t,
                                                  const int64_t* __restrict__ off, int64_t nseg,
                                                  const double* __restrict__ scale, int64_t ntot,
                                                  int64_t* __restrict__ tsum,
                                                  int32_t* __restrict__ status) {
  __shared__ int ws[FT / 32];
  const int64_t tile = blockIdx.x;
  int cnt = 0;
  bool bad = false;
  int64_t seg = -1, sbeg = 0, send = 0;
  double sc = 0.0;
#pragma unroll
  for (int k = 0; k < FPT; ++k) {
    const int64_t e = tile * FTILE + k * FT + threadIdx.x;
    if (e < ntot && (seg < 0 || e >= send)) {
      seg = seg_of(off, nseg, e);
      sbeg = off[seg];
      send = off[seg + 1];
      sc = scale[seg];
    }
    T x;  // every lane takes part (the point's neighbours come by shuffles)
    cnt += fin_point<T, KIND>(src, t, e, ntot, sbeg, send, sc, &x, &bad);
  }
  if (bad) atomicOr(status, 1);
  int tot;
  block_exclusive_sum<FT>(cnt, ws, &tot);
  if (threadIdx.x == 0) tsum[tile] = tot;
}

template <typename T, int KIND>
__global__ void __launch_bounds__(FT, 4) k_fin_write(const void* __restrict__ src,
                                                  const T* __restrict__ t,
                                                  const int64_t* __restrict__ off, int64_t nseg,
                                                  const double* __restrict__ scale, int64_t ntot,
                                                  const int64_t* __restrict__ tbase,
                                                  T* __restrict__ t_out, T* __restrict__ v_out,
                                                  int64_t* __restrict__ off_out) {
  constexpr int NW = FT / 32;
  __shared__ int s_cnt[FPT * NW];
  __shared__ int s_tot;
  __shared__ T s_t[FTILE], s_v[FTILE];
  const int64_t tile = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T val[FPT];
  uint32_t keep = 0, start = 0, ball[FPT];
  int64_t sstart[FPT];
  bool bad = false;
  int64_t seg = -1, sbeg = 0, send = 0;
  double sc = 0.0;
#pragma unroll
  for (int k = 0; k < FPT; ++k) {
    const int64_t e = tile * FTILE + k * FT + threadIdx.x;
    if (e < ntot && (seg < 0 || e >= send)) {
      seg = seg_of(off, nseg, e);
      sbeg = off[seg];
      send = off[seg + 1];
      sc = scale[seg];
    }
    const bool kp = fin_point<T, KIND>(src, t, e, ntot, sbeg, send, sc, &val[k], &bad);
    if (e < ntot && sbeg == e) {  // e starts node seg (and every empty node just before it)
      start |= 1u << k;
      sstart[k] = seg;
    }
    keep |= (uint32_t)kp << k;
  }
  // ballots after all the points' loads are in flight (a ballot per point would make every
  // point's loads wait for the previous point's)
#pragma unroll
  for (int k = 0; k < FPT; ++k) {
    ball[k] = __ballot_sync(0xffffffffu, (keep >> k) & 1u);
    if (lane == 0) s_cnt[k * NW + w] = __popc(ball[k]);
  }
  __syncthreads();
  if (w == 0) {  // exclusive scan of the FPT * NW warp counts in point order
    int run = 0;
    for (int base = 0; base < FPT * NW; base += 32) {
      const int x = base + lane < FPT * NW ? s_cnt[base + lane] : 0;
      int inc = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (base + lane < FPT * NW) s_cnt[base + lane] = run + inc - x;
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) s_tot = run;
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < FPT; ++k) {
    const int64_t e = tile * FTILE + k * FT + threadIdx.x;
    const int r = s_cnt[k * NW + w] + __popc(ball[k] & lt);
    if ((keep >> k) & 1u) {
      s_t[r] = t[e];
      s_v[r] = val[k];
    }
    // a node starting at point e: its output offset is the kept count before e
    if ((start >> k) & 1u)
      for (int64_t q = sstart[k]; q >= 0 && off[q] == e; --q) off_out[q] = tbase[tile] + r;
  }
  const int tot = s_tot;
  if (tile == gridDim.x - 1 && threadIdx.x == 0)  // the end, and nodes that start there
    for (int64_t q = nseg; q >= 0 && off[q] >= ntot; --q) off_out[q] = tbase[tile] + tot;
  __syncthreads();
  const int64_t ob = tbase[tile];
  for (int x = threadIdx.x; x < tot; x += FT) {
    t_out[ob + x] = s_t[x];
    v_out[ob + x] = s_v[x];
  }
}

// single-CTA exclusive scan of n int64 counts -> out[0..n]
__global__ void __launch_bounds__(1024) k_scan_counts(const int64_t* __restrict__ in, int64_t n,
                                                      int64_t* __restrict__ out) {
  __shared__ int64_t wsum[32];
  const int tid = threadIdx.x;
  const int64_t per = (n + 1023) / 1024;
  const int64_t b = min((int64_t)tid * per, n), e = min(b + per, n);
  int64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += in[i];
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

// flag counts per tile of FTILE points (for pcf_compact)
__global__ void __launch_bounds__(FT) k_flag_count(const int32_t* __restrict__ flag,
                                                   int64_t ntot, int64_t* __restrict__ tsum) {
  __shared__ int ws[FT / 32];
  const int64_t e0 = blockIdx.x * (int64_t)FTILE + threadIdx.x * FPT;
  int c = 0;
  for (int q = 0; q < FPT; ++q)
    if (e0 + q < ntot) c += flag[e0 + q] != 0;
  int tot;
  block_exclusive_sum<FT>(c, ws, &tot);
  if (threadIdx.x == 0) tsum[blockIdx.x] = tot;
}

// positions of the flagged points (exclusive scan within the tile + the tile base)
__global__ void __launch_bounds__(FT) k_flag_pos(const int32_t* __restrict__ flag, int64_t ntot,
                                                 const int64_t* __restrict__ tbase,
                                                 int64_t* __restrict__ pos) {
  __shared__ int ws[FT / 32];
  const int64_t e0 = blockIdx.x * (int64_t)FTILE + threadIdx.x * FPT;
  int c = 0;
  for (int q = 0; q < FPT; ++q)
    if (e0 + q < ntot) c += flag[e0 + q] != 0;
  int tot;
  int64_t p = tbase[blockIdx.x] + block_exclusive_sum<FT>(c, ws, &tot);
  for (int q = 0; q < FPT; ++q)
    if (e0 + q < ntot) {
      pos[e0 + q] = p;
      p += flag[e0 + q] != 0;
    }
}

static int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace pcfb

using namespace pcfb;

extern "C" {

int pcf_scan_workspace(int64_t ntot, int64_t* bytes) {
  const int64_t nt = (ntot > 0 ? ntot : 1) / FTILE + 1;
  *bytes = 2 * (nt + 1) * (int64_t)sizeof(int64_t);
  return PCF_OK;
}

// Exclusive scan of flags -> positions, scatter kept points, output node offsets.
// value_bytes: 4 or 8 (element size of sv/sv2), time_bytes: 4 or 8.  sv2 may be NULL.
int pcf_compact(int is_f32, const void* st_dev, const void* sv_dev, const void* sv2_dev,
                int value_bytes, const int32_t* flag_dev, int64_t ntot, const int64_t* off_in_dev,
                const int64_t* src_dev, int64_t nout, int64_t* pos_dev, void* temp_dev,
                int64_t temp_bytes, void* t_out_dev, void* v_out_dev, void* v2_out_dev,
                int64_t* off_out_dev, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (ntot > 0) {
    int64_t need = 0;
    pcf_scan_workspace(ntot, &need);
    if (!temp_dev || temp_bytes < need) {
      set_error("pcf_compact: workspace %lld < %lld bytes", (long long)temp_bytes,
                (long long)need);
      return PCF_ERR_ARG;
    }
    const int64_t nt = (ntot + FTILE - 1) / FTILE;
    int64_t* tsum = (int64_t*)temp_dev;
    int64_t* tbase = tsum + (nt + 1);
    k_flag_count<<<(unsigned)nt, FT, 0, s>>>(flag_dev, ntot, tsum);
    k_scan_counts<<<1, 1024, 0, s>>>(tsum, nt, tbase);
    k_flag_pos<<<(unsigned)nt, FT, 0, s>>>(flag_dev, ntot, tbase, pos_dev);
    const int g = grid_for(ntot, 256);
    if (is_f32 && value_bytes == 4)
      k_scatter<float, float><<<g, 256, 0, s>>>((const float*)st_dev, (const float*)sv_dev,
                                                (const float*)sv2_dev, flag_dev, pos_dev, ntot,
                                                (float*)t_out_dev, (float*)v_out_dev,
                                                (float*)v2_out_dev);
    else if (is_f32)
      k_scatter<float, double><<<g, 256, 0, s>>>((const float*)st_dev, (const double*)sv_dev,
                                                 (const double*)sv2_dev, flag_dev, pos_dev, ntot,
                                                 (float*)t_out_dev, (double*)v_out_dev,
                                                 (double*)v2_out_dev);
    else
      k_scatter<double, double><<<g, 256, 0, s>>>((const double*)st_dev, (const double*)sv_dev,
                                                  (const double*)sv2_dev, flag_dev, pos_dev, ntot,
                                                  (double*)t_out_dev, (double*)v_out_dev,
                                                  (double*)v2_out_dev);
  }
  k_out_offsets<<<grid_for(nout + 1, 256), 256, 0, s>>>(off_in_dev, src_dev, nout, pos_dev,
                                                         flag_dev, ntot, off_out_dev);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("pcf_compact: %s", cudaGetErrorString(e));
    return PCF_ERR_CUDA;
  }
  return PCF_OK;
}

int pcf_scale_flag(int is_f32, const void* v_dev, const void* t_dev, const int64_t* off_dev,
                   int64_t nseg, const double* scale_dev, int64_t ntot, void* sv_dev,
                   int32_t* flag_dev, int32_t* status_dev, void* stream) {
  if (ntot <= 0) return PCF_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int g = grid_for(ntot, 256);
  if (is_f32)
    k_scale_flag<float><<<g, 256, 0, s>>>((const float*)v_dev, (const float*)t_dev, off_dev, nseg,
                                          scale_dev, ntot, (float*)sv_dev, flag_dev, status_dev);
  else
    k_scale_flag<double><<<g, 256, 0, s>>>((const double*)v_dev, (const double*)t_dev, off_dev,
                                           nseg, scale_dev, ntot, (double*)sv_dev, flag_dev,
                                           status_dev);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("pcf_scale_flag: %s", cudaGetErrorString(e));
    return PCF_ERR_CUDA;
  }
  return PCF_OK;
}

int pcf_std_flag(int is_f32, int take_sqrt, const double* m2_dev, const void* t_dev,
                 const int64_t* off_dev, int64_t nseg, const double* scale_dev, int64_t ntot,
                 void* sv_dev, int32_t* flag_dev, int32_t* status_dev, void* stream) {
  if (ntot <= 0) return PCF_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int g = grid_for(ntot, 256);
#define PCF_SF(T, SQ)                                                                      \
  k_std_flag<T, SQ><<<g, 256, 0, s>>>(m2_dev, (const T*)t_dev, off_dev, nseg, scale_dev, ntot, \
                                      (T*)sv_dev, flag_dev, status_dev)
  if (is_f32) {
    if (take_sqrt) PCF_SF(float, true); else PCF_SF(float, false);
  } else {
    if (take_sqrt) PCF_SF(double, true); else PCF_SF(double, false);
  }
#undef PCF_SF
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("pcf_std_flag: %s", cudaGetErrorString(e));
    return PCF_ERR_CUDA;
  }
  return PCF_OK;
}


int pcf_finalize_workspace(int64_t ntot, int64_t* bytes) {
  if (!bytes || ntot < 0) {
    set_error("pcf_finalize_workspace: bad arguments");
    return PCF_ERR_ARG;
  }
  const int64_t nt = (ntot > 0 ? ntot : 1) / FTILE + 1;
  *bytes = 2 * (nt + 1) * (int64_t)sizeof(int64_t);
  return PCF_OK;
}

int pcf_finalize(int kind, int is_f32, const void* src_dev, const void* t_dev,
                 const int64_t* off_dev, int64_t nseg, const double* scale_dev, int64_t ntot,
                 void* t_out_dev, void* v_out_dev, int64_t* off_out_dev, int32_t* status_dev,
                 void* ws_dev, int64_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (kind < 0 || kind > 2 || nseg < 1 || ntot < 0 || !src_dev || !t_dev || !off_dev || !scale_dev ||
      !t_out_dev || !v_out_dev || !off_out_dev || !status_dev) {
    set_error("pcf_finalize: bad arguments");
    return PCF_ERR_ARG;
  }
  if (ntot == 0) {
    cudaError_t e = cudaMemsetAsync(off_out_dev, 0, (nseg + 1) * sizeof(int64_t), s);
    return e == cudaSuccess ? PCF_OK : (set_error("pcf_finalize: %s", cudaGetErrorString(e)), PCF_ERR_CUDA);
  }
  int64_t need = 0;
  pcf_finalize_workspace(ntot, &need);
  if (!ws_dev || ws_bytes < need) {
    set_error("pcf_finalize: workspace %lld < %lld bytes", (long long)ws_bytes, (long long)need);
    return PCF_ERR_ARG;
  }
  const int64_t nt = (ntot + FTILE - 1) / FTILE;
  int64_t* tsum = (int64_t*)ws_dev;
  int64_t* tbase = tsum + (nt + 1);
#define PCF_FIN(T, KD)                                                                        \
  do {                                                                                        \
    cudaFuncSetAttribute(k_fin_write<T, KD>, cudaFuncAttributePreferredSharedMemoryCarveout,   \
                         cudaSharedmemCarveoutMaxShared);                                     \
    k_fin_count<T, KD><<<(unsigned)nt, FT, 0, s>>>(src_dev, (const T*)t_dev, off_dev, nseg,   \
                                                   scale_dev, ntot, tsum, status_dev);       \
    k_scan_counts<<<1, 1024, 0, s>>>(tsum, nt, tbase);                                        \
    k_fin_write<T, KD><<<(unsigned)nt, FT, 0, s>>>(src_dev, (const T*)t_dev, off_dev, nseg,   \
                                                   scale_dev, ntot, tbase, (T*)t_out_dev,    \
                                                   (T*)v_out_dev, off_out_dev);              \
  } while (0)
  if (is_f32) {
    if (kind == 0) PCF_FIN(float, 0); else if (kind == 1) PCF_FIN(float, 1); else PCF_FIN(float, 2);
  } else {
    if (kind == 0) PCF_FIN(double, 0); else if (kind == 1) PCF_FIN(double, 1); else PCF_FIN(double, 2);
  }
#undef PCF_FIN
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("pcf_finalize: %s", cudaGetErrorString(e));
    return PCF_ERR_CUDA;
  }
  return PCF_OK;
}

}  // extern "C"
