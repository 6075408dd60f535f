// Reduction path helpers: compaction (scan + scatter) and the mean/std finalisation
// (reduce.py:211-238, core.py:165-214).  The tree levels themselves are in pcf_level.cu.
//
// The finalisation flags every point of the root node(s) -- keep where the scaled value
// differs from the previous surviving point's (minimize_discretization), drop zero-width
// pieces left by non-compacting levels -- and pcf_compact turns the flags into positions
// (device exclusive scan) and scatters the kept points and the node offsets.
#define CCCL_IGNORE_DEPRECATED_API 1
#include <cub/cub.cuh>
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

}  // extern "C"
