// Reduction path: one level of the fixed binary reduction tree of reduce.tree_reduce
// (pkg/src/pcflib/reduce.py:189-208), the pointwise combination of reduce_pair
// (reduce.py:31-63), the mean/std finalisation (reduce.py:211-238, core.py:165-214), and
// the parallel-moments (Chan) combination used for std.
//
// A level is a list of nodes (PCFs as SoA times/values + int64 offsets).  Output node k
// merges input nodes src[k] and src[k]+1 (cnt[k] == 2) or passes src[k] through
// (cnt[k] == 1, the reference's "No-Op passthrough").  Because output nodes consume
// consecutive input nodes, the merged candidate sequence of output node k occupies
// exactly the input positions [off[src[k]], off[src[k]+cnt[k]]): K5 writes one
// candidate (time, value, keep flag) per input point in place of that range, a device
// scan turns flags into output positions, and K5c scatters the kept points.  The keep
// rule reproduces reduce_pair's emission: a point at every distinct breakpoint whose
// combined value differs from the value of the cell just before it (equivalently, from
// the last emitted value), the t = 0 point always.
#define CCCL_IGNORE_DEPRECATED_API 1
#include <cub/cub.cuh>
#include "pcf_common.cuh"
#include "pcf_internal.h"

namespace pcfb {

enum ROp { R_ADD = 0, R_MAX = 1, R_MIN = 2, R_MUL = 3 };

template <int OP>
__device__ __forceinline__ double rop(double x, double y) {
  if (OP == R_ADD) return __dadd_rn(x, y);
  if (OP == R_MUL) return __dmul_rn(x, y);
  if (OP == R_MAX) return x > y ? x : y;  // Python max(x, y): first arg unless y > x
  return y < x ? y : x;                    // Python min(x, y)
}

template <typename T> __device__ __forceinline__ T to_t(double x);
template <> __device__ __forceinline__ double to_t<double>(double x) { return x; }
template <> __device__ __forceinline__ float to_t<float>(double x) { return __double2float_rn(x); }

constexpr int kChunk = 16;  // candidate positions per thread

// Locate the output node whose candidate range contains global position e:
// largest k in [0, nout) with off[src[k]] <= e.
__device__ __forceinline__ int64_t find_node(const int64_t* __restrict__ off,
                                             const int64_t* __restrict__ src, int64_t nout,
                                             int64_t e) {
  int64_t lo = 0, hi = nout - 1;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) >> 1;
    if (off[src[mid]] <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Co-rank on the stable merge of A (times ta, na) and B (tb, nb), A first on ties:
// number of A elements among the first m merged elements.
template <typename T>
__device__ __forceinline__ int64_t corank(const T* __restrict__ ta, int64_t na,
                                          const T* __restrict__ tb, int64_t nb, int64_t m) {
  int64_t lo = m > nb ? m - nb : 0, hi = m < na ? m : na;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (ta[mid] <= tb[m - mid - 1]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// For a merge position m > 0 with co-rank (i, j): index of the B piece active at the time
// T of position m-1 (T = max(ta[i-1], tb[j-1]); B[j] counts too when it ties with T).
// The A piece active at T is always i-1 (A times are strictly increasing).
template <typename T>
__device__ __forceinline__ int64_t prev_cell_b(const T* __restrict__ ta, const T* __restrict__ tb,
                                               int64_t nb, int64_t i, int64_t j) {
  const T tp = (j > 0 && tb[j - 1] > ta[i - 1]) ? tb[j - 1] : ta[i - 1];
  return j + ((j < nb && tb[j] == tp) ? 1 : 0) - 1;
}

// ------------------------------------------------------------------ K5: value combine
template <typename T, int OP>
__global__ void k_level_merge(const T* __restrict__ t, const T* __restrict__ v,
                              const int64_t* __restrict__ off, const int64_t* __restrict__ src,
                              const int32_t* __restrict__ cnt, int64_t nout, int64_t ntot,
                              T* __restrict__ st, T* __restrict__ sv, int32_t* __restrict__ flag,
                              int32_t* __restrict__ status) {
  const int64_t nchunks = (ntot + kChunk - 1) / kChunk;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nchunks;
       c += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = c * kChunk;
    const int64_t e1 = min(e + kChunk, ntot);
    while (e < e1) {
      const int64_t k = find_node(off, src, nout, e);
      const int64_t s = src[k];
      const int64_t base = off[s];
      if (cnt[k] == 1) {  // passthrough: points kept verbatim (reduce.py:205-206)
        const int64_t end = min(e1, off[s + 1]);
        for (; e < end; ++e) {
          st[e] = t[e];
          sv[e] = v[e];
          flag[e] = 1;
        }
        continue;
      }
      const T* ta = t + base;
      const T* va = v + base;
      const int64_t na = off[s + 1] - base;
      const T* tb = t + off[s + 1];
      const T* vb = v + off[s + 1];
      const int64_t nb = off[s + 2] - off[s + 1];
      int64_t m = e - base;
      const int64_t mend = min(e1 - base, na + nb);
      int64_t i = corank(ta, na, tb, nb, m);
      int64_t j = m - i;
      // value of the cell at the time of position m-1 (defined when m > 0)
      T prev = T(0);
      if (m > 0) {
        const int64_t jt = prev_cell_b(ta, tb, nb, i, j);
        prev = to_t<T>(rop<OP>((double)va[i - 1], (double)vb[jt]));
      }
      for (; m < mend; ++m, ++e) {
        const bool takeA = (i < na) && (j >= nb || ta[i] <= tb[j]);
        T tt, val;
        int32_t keep;
        if (takeA) {
          tt = ta[i];
          const int64_t jb = j + ((j < nb && tb[j] == tt) ? 1 : 0) - 1;
          val = to_t<T>(rop<OP>((double)va[i], (double)vb[jb]));
          keep = (m == 0) || (val != prev);
          prev = val;
          ++i;
        } else {
          tt = tb[j];
          const bool dup = (i > 0 && ta[i - 1] == tt);
          if (dup) {
            val = prev;
            keep = 0;
          } else {
            val = to_t<T>(rop<OP>((double)va[i - 1], (double)vb[j]));
            keep = (val != prev);
            prev = val;
          }
          ++j;
        }
        if (keep && !isfinite((double)val)) atomicOr(status, 1);
        st[e] = tt;
        sv[e] = val;
        flag[e] = keep;
      }
    }
  }
}

// ------------------------------------------------------- K7: parallel moments (Chan)
// Node state per cell: (mean, M2) over the node's n leaves.  Merging A (nA leaves) and
// B (nB): d = mB - mA, n = nA + nB, mean = mA + d*nB/n, M2 = M2A + M2B + d^2*nA*nB/n.
// Leaves: mean = value, M2 = 0.  Points are kept where (mean, M2) changes.
template <typename T>
__global__ void k_level_moments(const T* __restrict__ t, const double* __restrict__ mu,
                                const double* __restrict__ m2, const int64_t* __restrict__ off,
                                const int64_t* __restrict__ src, const int32_t* __restrict__ cnt,
                                const int64_t* __restrict__ leaves, int64_t nout, int64_t ntot,
                                T* __restrict__ st, double* __restrict__ smu,
                                double* __restrict__ sm2, int32_t* __restrict__ flag) {
  const int64_t nchunks = (ntot + kChunk - 1) / kChunk;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nchunks;
       c += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = c * kChunk;
    const int64_t e1 = min(e + kChunk, ntot);
    while (e < e1) {
      const int64_t k = find_node(off, src, nout, e);
      const int64_t s = src[k];
      const int64_t base = off[s];
      if (cnt[k] == 1) {
        const int64_t end = min(e1, off[s + 1]);
        for (; e < end; ++e) {
          st[e] = t[e];
          smu[e] = mu[e];
          sm2[e] = m2[e];
          flag[e] = 1;
        }
        continue;
      }
      const double nA = (double)leaves[s], nB = (double)leaves[s + 1];
      const double n = nA + nB;
      const double wB = nB / n, wAB = nA * nB / n;
      const T* ta = t + base;
      const int64_t na = off[s + 1] - base;
      const T* tb = t + off[s + 1];
      const int64_t nb = off[s + 2] - off[s + 1];
      const double* mua = mu + base;
      const double* m2a = m2 + base;
      const double* mub = mu + off[s + 1];
      const double* m2b = m2 + off[s + 1];
      auto comb = [&](int64_t ia, int64_t ib, double& om, double& o2) {
        const double d = mub[ib] - mua[ia];
        om = mua[ia] + d * wB;
        o2 = (m2a[ia] + m2b[ib]) + d * d * wAB;
      };
      int64_t m = e - base;
      const int64_t mend = min(e1 - base, na + nb);
      int64_t i = corank(ta, na, tb, nb, m);
      int64_t j = m - i;
      double pm = 0.0, p2 = 0.0;
      if (m > 0) comb(i - 1, prev_cell_b(ta, tb, nb, i, j), pm, p2);
      for (; m < mend; ++m, ++e) {
        const bool takeA = (i < na) && (j >= nb || ta[i] <= tb[j]);
        T tt;
        double om = pm, o2 = p2;
        int32_t keep = 0;
        if (takeA) {
          tt = ta[i];
          const int64_t jb = j + ((j < nb && tb[j] == tt) ? 1 : 0) - 1;
          comb(i, jb, om, o2);
          keep = (m == 0) || om != pm || o2 != p2;
          pm = om;
          p2 = o2;
          ++i;
        } else {
          tt = tb[j];
          const bool dup = (i > 0 && ta[i - 1] == tt);
          if (!dup) {
            comb(i - 1, j, om, o2);
            keep = om != pm || o2 != p2;
            pm = om;
            p2 = o2;
          }
          ++j;
        }
        st[e] = tt;
        smu[e] = om;
        sm2[e] = o2;
        flag[e] = keep;
      }
    }
  }
}

// ------------------------------------------------------------ compaction (K5c)
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
template <typename T>
__global__ void k_scale_flag(const T* __restrict__ v, const int64_t* __restrict__ off,
                             int64_t nseg, const double* __restrict__ scale, int64_t ntot,
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
    if (!isfinite((double)x)) atomicOr(status, 1);
    if (e == off[lo]) {
      flag[e] = 1;
    } else {
      const T y = v[e - 1] * a;
      flag[e] = (x != y);
    }
  }
}

// std: s = T(sqrt(double(T(M2 * scale)))) (variance scale in float64, then
// core.apply_unary(math.sqrt)), keep where s changes.
template <typename T, bool SQRT>
__global__ void k_std_flag(const double* __restrict__ m2, const int64_t* __restrict__ off,
                           int64_t nseg, const double* __restrict__ scale, int64_t ntot,
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
    if (!isfinite((double)x)) atomicOr(status, 1);
    flag[e] = (e == off[lo]) ? 1 : (x != sd(e - 1));
  }
}

struct Widen {
  __host__ __device__ __forceinline__ int64_t operator()(int32_t x) const { return (int64_t)x; }
};

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
  size_t b = 0;
  cub::TransformInputIterator<int64_t, Widen, const int32_t*> it(nullptr, Widen());
  cub::DeviceScan::ExclusiveSum(nullptr, b, it, (int64_t*)nullptr,
                                (int64_t)(ntot > 0 ? ntot : 1));
  *bytes = (int64_t)b;
  return PCF_OK;
}

int pcf_level_merge(int op, int is_f32, const void* t_dev, const void* v_dev,
                    const int64_t* off_dev, const int64_t* src_dev, const int32_t* cnt_dev,
                    int64_t nout, int64_t ntot, void* st_dev, void* sv_dev, int32_t* flag_dev,
                    int32_t* status_dev, void* stream) {
  if (ntot <= 0 || nout <= 0) return PCF_OK;
  if (op < 0 || op > 3 || !t_dev || !v_dev || !off_dev || !src_dev || !cnt_dev || !st_dev ||
      !sv_dev || !flag_dev || !status_dev) {
    set_error("pcf_level_merge: bad arguments");
    return PCF_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int th = 256;
  const int g = grid_for((ntot + kChunk - 1) / kChunk, th);
#define PCF_LM(T, OP)                                                                       \
  k_level_merge<T, OP><<<g, th, 0, s>>>((const T*)t_dev, (const T*)v_dev, off_dev, src_dev, \
                                        cnt_dev, nout, ntot, (T*)st_dev, (T*)sv_dev, flag_dev, \
                                        status_dev)
  if (is_f32) {
    switch (op) {
      case R_ADD: PCF_LM(float, R_ADD); break;
      case R_MAX: PCF_LM(float, R_MAX); break;
      case R_MIN: PCF_LM(float, R_MIN); break;
      default: PCF_LM(float, R_MUL); break;
    }
  } else {
    switch (op) {
      case R_ADD: PCF_LM(double, R_ADD); break;
      case R_MAX: PCF_LM(double, R_MAX); break;
      case R_MIN: PCF_LM(double, R_MIN); break;
      default: PCF_LM(double, R_MUL); break;
    }
  }
#undef PCF_LM
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("pcf_level_merge: %s", cudaGetErrorString(e));
    return PCF_ERR_CUDA;
  }
  return PCF_OK;
}

int pcf_level_moments(int is_f32, const void* t_dev, const double* mu_dev, const double* m2_dev,
                      const int64_t* off_dev, const int64_t* src_dev, const int32_t* cnt_dev,
                      const int64_t* leaves_dev, int64_t nout, int64_t ntot, void* st_dev,
                      double* smu_dev, double* sm2_dev, int32_t* flag_dev, void* stream) {
  if (ntot <= 0 || nout <= 0) return PCF_OK;
  if (!t_dev || !mu_dev || !m2_dev || !off_dev || !src_dev || !cnt_dev || !leaves_dev ||
      !st_dev || !smu_dev || !sm2_dev || !flag_dev) {
    set_error("pcf_level_moments: bad arguments");
    return PCF_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int th = 256;
  const int g = grid_for((ntot + kChunk - 1) / kChunk, th);
  if (is_f32)
    k_level_moments<float><<<g, th, 0, s>>>((const float*)t_dev, mu_dev, m2_dev, off_dev, src_dev,
                                            cnt_dev, leaves_dev, nout, ntot, (float*)st_dev,
                                            smu_dev, sm2_dev, flag_dev);
  else
    k_level_moments<double><<<g, th, 0, s>>>((const double*)t_dev, mu_dev, m2_dev, off_dev,
                                             src_dev, cnt_dev, leaves_dev, nout, ntot,
                                             (double*)st_dev, smu_dev, sm2_dev, flag_dev);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("pcf_level_moments: %s", cudaGetErrorString(e));
    return PCF_ERR_CUDA;
  }
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
    size_t tb = (size_t)temp_bytes;
    cub::TransformInputIterator<int64_t, Widen, const int32_t*> it(flag_dev, Widen());
    cudaError_t e = cub::DeviceScan::ExclusiveSum(temp_dev, tb, it, pos_dev, (int64_t)ntot, s);
    if (e != cudaSuccess) {
      set_error("pcf_compact scan: %s", cudaGetErrorString(e));
      return PCF_ERR_CUDA;
    }
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

int pcf_scale_flag(int is_f32, const void* v_dev, const int64_t* off_dev, int64_t nseg,
                   const double* scale_dev, int64_t ntot, void* sv_dev, int32_t* flag_dev,
                   int32_t* status_dev, void* stream) {
  if (ntot <= 0) return PCF_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int g = grid_for(ntot, 256);
  if (is_f32)
    k_scale_flag<float><<<g, 256, 0, s>>>((const float*)v_dev, off_dev, nseg, scale_dev, ntot,
                                          (float*)sv_dev, flag_dev, status_dev);
  else
    k_scale_flag<double><<<g, 256, 0, s>>>((const double*)v_dev, off_dev, nseg, scale_dev, ntot,
                                           (double*)sv_dev, flag_dev, status_dev);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("pcf_scale_flag: %s", cudaGetErrorString(e));
    return PCF_ERR_CUDA;
  }
  return PCF_OK;
}

int pcf_std_flag(int is_f32, int take_sqrt, const double* m2_dev, const int64_t* off_dev,
                 int64_t nseg, const double* scale_dev, int64_t ntot, void* sv_dev,
                 int32_t* flag_dev, int32_t* status_dev, void* stream) {
  if (ntot <= 0) return PCF_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int g = grid_for(ntot, 256);
#define PCF_SF(T, SQ)                                                                      \
  k_std_flag<T, SQ><<<g, 256, 0, s>>>(m2_dev, off_dev, nseg, scale_dev, ntot, (T*)sv_dev, \
                                      flag_dev, status_dev)
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

}  // extern "C"
