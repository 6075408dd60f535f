// Shared device helpers for the B200 rectangle-iteration engine.
//
// Data layout (HBM): every PCF f with stored rows (t_0=0, v_0) .. (t_{n-1}, v_{n-1})
// is stored as n 16-byte "records"  rec[k] = (t_next = t_{k+1}, v = v_k), with
// t_next = +inf for the last record.  A record is exactly what one step of the
// reference sweep (_sweepkern.pyx:38-41) reads for one cursor: the value on the
// current piece and the time at which that piece ends.  Collections are stored
// size-sorted (descending) and concatenated, so any run of consecutive PCFs is one
// contiguous byte range -> one cp.async.bulk copy.
#pragma once
#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#else  // NVRTC (user integrands, pcf_jit.cu): no host headers
typedef long long int64_t;
typedef unsigned long long uint64_t;
typedef int int32_t;
typedef unsigned int uint32_t;
#ifndef INFINITY
#define INFINITY __int_as_float(0x7f800000)
#endif
#endif

#ifndef __CUDACC_RTC__
#include "pcf_pow.cuh"  // libm-exact pow (glibc 2.39 restated; tables from libm.so.6)
#endif

namespace pcfb {

struct __align__(16) Rec {
  double t;  // end of this piece (= next breakpoint), +inf on the last piece
  double v;  // value on this piece
};

// 8-byte record for float32 collections (the reference widens every operand to float64
// before any arithmetic, pyx:38-41; so do the kernels, after the shared-memory load).
struct __align__(8) Rec32 {
  float t;
  float v;
};

// Integrand kinds.  OP_LP: p = 1 is |x - y| (pow(d, 1.0) == d exactly); any other p is
// H_LPX = pow(|x - y|, p) with the C library's pow restated bit for bit (pcf_pow.cuh), as
// the reference computes every cell (pyx:43-46).  PCF_OP_FAST_POW (fast plan) trades that
// for d*d (H_L2), d*d*|d| (H_L3) or CUDA's pow (H_LP): within 1 ulp per cell, rel 1e-12
// per entry.  OP_INNER is v_f * v_g.
enum HKind { H_L1 = 0, H_L2 = 1, H_L3 = 2, H_LP = 3, H_INNER = 4, H_USER = 5, H_LPX = 6 };

// A user integrand compiled at run time (pcf_jit.cu defines it; never referenced by the
// nvcc-built kernels, where HK is one of the op codes above).
__device__ double pcf_user_h(double x, double y);
__device__ double pcf_user_r(double x);

// h(v_f, v_g): _sweepkern.pyx:43-46.  Rounded ops only (no FMA contraction) so the
// p=1 and inner-product paths reproduce the gcc -O2 (SSE2, no FMA) reference bitwise.
template <int HK>
__device__ __forceinline__ double hval(double x, double y, double p) {
  if (HK == H_L1) return fabs(__dsub_rn(x, y));
  if (HK == H_L2) {
    double d = __dsub_rn(x, y);
    return __dmul_rn(d, d);
  }
  if (HK == H_L3) {
    double d = fabs(__dsub_rn(x, y));
    return __dmul_rn(__dmul_rn(d, d), d);
  }
  if (HK == H_LP) return pow(fabs(__dsub_rn(x, y)), p);
#ifndef __CUDACC_RTC__
  if constexpr (HK == H_LPX) return pcfpow::pow(fabs(__dsub_rn(x, y)), p);
#endif
  if constexpr (HK == H_USER) return pcf_user_h(x, y);
  return __dmul_rn(x, y);
}

// ---------------------------------------------------------------- mbarrier / bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

// tx-count increment without an arrival (several threads register their bulk copies,
// one thread arrives afterwards)
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 1-D bulk async copy global -> shared (TMA engine, SASS UBLKCP), completion
// counted in bytes on `bar`.  bytes must be a multiple of 16, both addresses 16B
// aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Bulk prefetch of a global byte range into L2 (no completion tracking): warms the next
// column chunk while the current one is walked, so its later bulk copy hits L2.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// ------------------------------------------------- per-thread async copies (LDGSTS)
// One record global -> shared, completion tracked by the issuing thread's commit groups.
// 16-byte records bypass L1 (.cg); 8-byte records must use .ca.
template <int BYTES, bool L1 = false>
__device__ __forceinline__ void cp_async_rec(uint32_t dst, const void* src) {
  if constexpr (BYTES == 16 && L1) {  // cached in L1: the rest of the 128-byte line is reused
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
  } else if constexpr (BYTES == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
  } else if constexpr (BYTES == 8) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
  }
}

__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// one record from a 32-bit shared-memory address
__device__ __forceinline__ void lds_rec(uint32_t a, double& t, double& v) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(t), "=d"(v) : "r"(a));
}
__device__ __forceinline__ void lds_rec(uint32_t a, float& t, float& v) {
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(t), "=f"(v) : "r"(a));
}

__device__ __forceinline__ uint32_t dynamic_smem_bytes() {
  uint32_t n;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(n));
  return n;
}

// Exclusive prefix sum of one int per thread over a CTA of NT threads (NT a multiple of 32,
// at most 1024); ws = shared scratch of NT / 32 ints.  Returns the thread's prefix and the
// CTA total in *total.  Ends with a barrier, so ws may be reused right after.
template <int NT>
__device__ __forceinline__ int block_exclusive_sum(int x, int* ws, int* total) {
  static_assert(NT % 32 == 0 && NT <= 1024, "block size");
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    int z = lane < NW ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    if (lane < NW) ws[lane] = z;
  }
  __syncthreads();
  const int before = w > 0 ? ws[w - 1] : 0;
  *total = ws[NW - 1];
  __syncthreads();
  return before + inc - x;
}

// Largest count of x in [0, n) with key(x) <= a, for sorted keys (upper_bound).
template <typename KeyF>
__device__ __forceinline__ int upper_bound_count(int n, double a, KeyF key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (key(mid) <= a) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// fill_block's root pow(acc, 1/p) (pyx:98,113-114) with the C library's pow, bit for bit
// (pow(x, 1.0) == x exactly, so p = 1 skips it)
__device__ __forceinline__ double root_p(double acc, double p) {
  if (p == 1.0) return acc;
#ifndef __CUDACC_RTC__
  return pcfpow::pow(acc, 1.0 / p);
#else
  return pow(acc, 1.0 / p);
#endif
}

template <typename T> __device__ __forceinline__ T cast_out(double x);
template <> __device__ __forceinline__ double cast_out<double>(double x) { return x; }
template <> __device__ __forceinline__ float cast_out<float>(double x) { return __double2float_rn(x); }

}  // namespace pcfb
